// Alg. 1: DFS over execution states; candidates are differences of
// two states (Theorem 1) with a unique sink (readings A3/A4), pruned as
// in P:626 ("too many operators ... or including multiple linear transformation
// primitives", reading A5/A18) and put in canonical order.
//
// Whole models are first partitioned (reading A17): cuts only at articulation
// tensors of the topological order, parts grown greedily to `partition_max` primitives,
// and Alg. 1 runs inside each part (a set inside one part is convex in G iff it is
// convex in the part, since a path that leaves a part never returns).
#include <functional>
#include "enumerate.h"

#include <algorithm>
#include <map>
#include <unordered_set>

#include "../../include/korch.h"

namespace korch {

namespace {
struct Dfs {
  int n;
  int64_t cap;
  std::vector<Bits> pred_bits;           // local indices
  std::unordered_set<Bits, BitsHash> B;  // database of execution states
  std::vector<Bits> order;               // insertion order (deterministic)
  Dfs(int nn, int64_t c) : n(nn), cap(c), pred_bits(nn) {}
  bool ready(const Bits& X, int v) const {  // forall (u,v) in E: u in X
    for (int i = 0; i < kMaxPrims / 64; ++i)
      if (pred_bits[v].w[i] & ~X.w[i]) return false;
    return true;
  }
  void run(const Bits& X) {  // Dfs(X), P:316-326 (iterative to bound stack depth)
    std::vector<Bits> stack{X};
    while (!stack.empty()) {
      Bits cur = stack.back();
      stack.pop_back();
      for (int v = n - 1; v >= 0; --v) {
        if (cur.test(v) || !ready(cur, v)) continue;
        Bits nx = cur;
        nx.set(v);
        if (B.insert(nx).second) {
          order.push_back(nx);
          if ((int64_t)B.size() > cap)
            throw KorchError(KORCH_E_STATE_EXPLOSION,
                             "more than " + std::to_string(cap) + " execution states");
          stack.push_back(nx);
        }
      }
    }
  }
};
}  // namespace

static std::vector<std::vector<int>> partition_k(const Graph& g, int max_nodes, int max_cross);

// Cuts where at most k tensors cross (all materialised), k = 1, 2, ... 8 until no part
// exceeds 2 * max_nodes (reading A17).
std::vector<std::vector<int>> partition_graph(const Graph& g, int max_nodes) {
  std::vector<std::vector<int>> parts;
  for (int k = 1; k <= 8; ++k) {
    parts = partition_k(g, max_nodes, k);
    size_t mx = 0;
    for (auto& p : parts) mx = std::max(mx, p.size());
    if ((int)mx <= 2 * max_nodes) break;
  }
  return parts;
}

static std::vector<std::vector<int>> partition_k(const Graph& g, int max_nodes, int max_cross) {
  int n = (int)g.prims.size();
  const std::vector<int>& topo = g.topo;
  std::vector<int> last_use(n, -1), ends(n + 1, 0);
  for (int i = 0; i < n; ++i)
    for (int w : g.succs[topo[i]]) last_use[i] = std::max(last_use[i], g.topo_index[w]);
  // cuts never split an operator's fission fragment (keeps operator-aligned kernels)
  std::map<long long, std::pair<int, int>> span;
  for (int i = 0; i < n; ++i) {
    int v = topo[i];
    long long op = g.prims[v].op_id >= 0 ? (long long)g.prims[v].op_id : -1LL - v;
    auto it = span.find(op);
    if (it == span.end()) span[op] = {i, i};
    else it->second = {std::min(it->second.first, i), std::max(it->second.second, i)};
  }
  std::vector<int> inside(n + 1, 0);
  for (auto& kv : span)
    if (kv.second.second > kv.second.first) {
      ++inside[kv.second.first];
      --inside[kv.second.second];
    }
  std::vector<char> cut_after(n, 0);
  int active = 0, open_ops = 0;
  for (int i = 0; i < n; ++i) {
    if (last_use[i] > i) {
      ++active;
      ++ends[last_use[i]];
    }
    active -= ends[i];
    open_ops += inside[i];
    cut_after[i] = active >= 1 && active <= max_cross && i < n - 1 && open_ops == 0;
  }
  std::vector<std::vector<int>> parts;
  int start = 0, last_cut = -1;
  for (int i = 0; i < n; ++i) {
    if (i - start + 1 > max_nodes && last_cut >= start) {
      parts.emplace_back(topo.begin() + start, topo.begin() + last_cut + 1);
      start = last_cut + 1;
      last_cut = -1;
      for (int j = start; j < i; ++j)
        if (cut_after[j]) last_cut = j;
    }
    if (cut_after[i]) last_cut = i;
  }
  parts.emplace_back(topo.begin() + start, topo.end());
  for (auto& p : parts) std::sort(p.begin(), p.end());
  return parts;
}

std::vector<Candidate> enumerate_candidates(const Graph& g, const EnumOpts& o, int64_t* n_states,
                                            std::vector<std::vector<int>>* parts_out) {
  int n = (int)g.prims.size();
  int pmax = o.partition_max > 0 ? o.partition_max : (n > kMaxPrims ? 64 : 0);
  std::vector<std::vector<int>> parts;
  if (pmax > 0) {
    parts = partition_graph(g, pmax);
  } else {
    parts.emplace_back();
    for (int v = 0; v < n; ++v) parts.back().push_back(v);
  }
  for (auto& p : parts)
    if ((int)p.size() > kMaxPrims)
      throw KorchError(KORCH_E_ARG, "a partition part has " + std::to_string(p.size()) +
                                        " primitives (> 256); no articulation tensor to cut at");
  std::vector<char> dense(n);
  for (int v = 0; v < n; ++v) dense[v] = g.is_dense_linear(v);
  std::vector<Candidate> out;
  int64_t total_states = 0;
  for (size_t pi = 0; pi < parts.size(); ++pi) {
    const std::vector<int>& part = parts[pi];
    int m = (int)part.size();
    std::vector<int> loc(n, -1);
    for (int i = 0; i < m; ++i) loc[part[i]] = i;
    Dfs d(m, o.max_states);
    std::vector<Bits> succ_bits(m);
    for (int i = 0; i < m; ++i) {
      for (int u : g.preds[part[i]])
        if (loc[u] >= 0) d.pred_bits[i].set(loc[u]);
      for (int w : g.succs[part[i]])
        if (loc[w] >= 0) succ_bits[i].set(loc[w]);
    }
    // descendants within the part (for the attention-pair rule, N2)
    std::vector<Bits> desc(m);
    if (o.attention_pairs) {
      std::vector<int> order_local;
      for (int v : g.topo)
        if (loc[v] >= 0) order_local.push_back(loc[v]);
      for (auto it = order_local.rbegin(); it != order_local.rend(); ++it) {
        int v = *it;
        for (int w : g.succs[part[v]])
          if (loc[w] >= 0) {
            desc[v].set(loc[w]);
            for (int i = 0; i < kMaxPrims / 64; ++i) desc[v].w[i] |= desc[loc[w]].w[i];
          }
      }
    }
    auto attention_ok = [&](const std::vector<int>& mem_local) {
      std::vector<int> lin;
      for (int v : mem_local)
        if (dense[part[v]]) lin.push_back(v);
      if (lin.size() != 2) return false;
      int a = lin[0], b = lin[1];
      if (g.topo_index[part[a]] > g.topo_index[part[b]]) std::swap(a, b);
      const Prim& pa = g.prims[part[a]];
      const Prim& pb = g.prims[part[b]];
      if (pa.kind != Kind::MatMul || pb.kind != Kind::MatMul) return false;
      auto feeds = [&](const Ref& r) {
        if (r.is_input || loc[r.id] < 0) return false;
        return loc[r.id] == a || desc[a].test(loc[r.id]);
      };
      return feeds(pb.in[0]) && !feeds(pb.in[1]);
    };
    Bits empty;
    d.B.insert(empty);  // reading A1: seed B with the empty state
    d.order.push_back(empty);
    d.run(empty);
    total_states += (int64_t)d.order.size();
    // for D1 subset D2: P' = D2 \ D1; keep unique-sink sets once.
    std::unordered_set<Bits, BitsHash> seen;
    const auto& S = d.order;
    for (size_t a = 0; a < S.size(); ++a) {
      for (size_t b = 0; b < S.size(); ++b) {
        if (!S[a].subset_of(S[b])) continue;
        Bits P = S[b].minus(S[a]);
        if (P.count() > o.max_prims) continue;
        if (!seen.insert(P).second) continue;
        int sink = -1, nsink = 0, nd = 0;
        std::vector<int> mem_local = P.list();
        for (int v : mem_local) {
          bool internal_succ = false;
          for (int i = 0; i < kMaxPrims / 64; ++i)
            if (succ_bits[v].w[i] & P.w[i]) { internal_succ = true; break; }
          if (!internal_succ) { sink = v; ++nsink; }
          nd += dense[part[v]];
        }
        if (nsink != 1) continue;                         // single output (A4)
        if (!o.keep_multi_linear && nd >= 2 &&            // P:626 (A18), relaxed for N2
            !(nd == 2 && o.attention_pairs && attention_ok(mem_local)))
          continue;
        Candidate c;
        for (int v : mem_local) c.members.push_back(part[v]);
        std::sort(c.members.begin(), c.members.end());
        c.output = part[sink];
        c.n_dense = nd;
        c.part = (int)pi;
        std::vector<int> ins, gins;
        std::vector<char> in_p(n, 0);
        for (int v : c.members) in_p[v] = 1;
        for (int v : c.members)
          for (auto& r : g.prims[v].in) {
            if (r.is_input) gins.push_back(r.id);
            else if (!in_p[r.id]) ins.push_back(r.id);
          }
        std::sort(ins.begin(), ins.end());
        ins.erase(std::unique(ins.begin(), ins.end()), ins.end());
        std::sort(gins.begin(), gins.end());
        gins.erase(std::unique(gins.begin(), gins.end()), gins.end());
        c.inputs = ins;
        c.graph_inputs = gins;
        out.push_back(std::move(c));
      }
    }
  }
  if (n_states) *n_states = total_states;
  if (parts_out) *parts_out = parts;
  // N1 ("for O in P'", P:352-360 possible output set; reading A32): every
  // single-output candidate (P', o) also yields (P', o, E) for each non-empty E of at most
  // max_outputs - 1 secondary outputs drawn from the members (other than o) that have a
  // consumer outside P' or are graph outputs (A3), with the shape of o
  if (o.max_outputs > 1) {
    std::vector<char> is_out(n, 0);
    for (int t : g.outputs) is_out[t] = 1;
    const size_t n_single = out.size();
    for (size_t ci = 0; ci < n_single; ++ci) {
      std::vector<char> in_p(n, 0);
      for (int v : out[ci].members) in_p[v] = 1;
      std::vector<int> xs;
      for (int u : out[ci].members) {
        if (u == out[ci].output || g.prims[u].shape != g.prims[out[ci].output].shape) continue;
        bool ext = is_out[u];
        for (int w : g.succs[u]) ext = ext || !in_p[w];
        if (ext) xs.push_back(u);
      }
      const int kmax = std::min<int>(o.max_outputs - 1, (int)xs.size());
      std::vector<int> pick;
      std::function<void(size_t)> rec = [&](size_t from) {
        if (!pick.empty()) {
          Candidate c = out[ci];
          c.extra_outputs = pick;
          out.push_back(std::move(c));
        }
        if ((int)pick.size() == kmax) return;
        for (size_t i = from; i < xs.size(); ++i) {
          pick.push_back(xs[i]);
          rec(i + 1);
          pick.pop_back();
        }
      };
      rec(0);
    }
  }
  std::sort(out.begin(), out.end(), [](const Candidate& x, const Candidate& y) {
    if (x.output != y.output) return x.output < y.output;
    if (x.members.size() != y.members.size()) return x.members.size() < y.members.size();
    if (x.members != y.members) return x.members < y.members;
    return x.extra_outputs < y.extra_outputs;
  });
  return out;
}

}  // namespace korch
