// Alg. 1: DFS over execution states; candidates are differences of
// two states (Theorem 1) with a unique sink (readings A3/A4), pruned as
// in P:626 ("too many operators ... or including multiple linear transformation
// primitives", reading A5/A18) and put in canonical order.
#include "enumerate.h"

#include <algorithm>
#include <unordered_set>

#include "../../include/korch.h"

namespace korch {

namespace {
struct Dfs {
  const Graph& g;
  int64_t cap;
  std::vector<Bits> pred_bits;
  std::unordered_set<Bits, BitsHash> B;  // database of execution states
  std::vector<Bits> order;               // insertion order (deterministic)
  Dfs(const Graph& gg, int64_t c) : g(gg), cap(c) {
    int n = (int)g.prims.size();
    pred_bits.resize(n);
    for (int v = 0; v < n; ++v)
      for (int u : g.preds[v]) pred_bits[v].set(u);
  }
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
      int n = (int)g.prims.size();
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

std::vector<Candidate> enumerate_candidates(const Graph& g, const EnumOpts& o, int64_t* n_states) {
  int n = (int)g.prims.size();
  if (n > kMaxPrims)
    throw KorchError(KORCH_E_ARG, "primitive graph has " + std::to_string(n) +
                                      " nodes; partition it to <= 256 first");
  Dfs d(g, o.max_states);
  Bits empty;
  d.B.insert(empty);  // reading A1: seed B with the empty state
  d.order.push_back(empty);
  d.run(empty);
  if (n_states) *n_states = (int64_t)d.order.size();

  std::vector<Bits> succ_bits(n);
  for (int v = 0; v < n; ++v)
    for (int w : g.succs[v]) succ_bits[v].set(w);
  std::vector<char> dense(n);
  for (int v = 0; v < n; ++v) dense[v] = g.is_dense_linear(v);

  // for D1 subset D2: P' = D2 \ D1; keep unique-sink sets once.
  std::unordered_set<Bits, BitsHash> seen;
  std::vector<Candidate> out;
  const auto& S = d.order;
  for (size_t a = 0; a < S.size(); ++a) {
    for (size_t b = 0; b < S.size(); ++b) {
      if (!S[a].subset_of(S[b])) continue;
      Bits P = S[b].minus(S[a]);
      int cnt = P.count();
      if (cnt > o.max_prims) continue;
      if (!seen.insert(P).second) continue;
      int sink = -1, nsink = 0, nd = 0;
      for (int v : P.list()) {
        bool internal_succ = false;
        for (int i = 0; i < kMaxPrims / 64; ++i)
          if (succ_bits[v].w[i] & P.w[i]) { internal_succ = true; break; }
        if (!internal_succ) { sink = v; ++nsink; }
        nd += dense[v];
      }
      if (nsink != 1) continue;                         // single output (A4)
      if (!o.keep_multi_linear && nd >= 2) continue;    // P:626 (A18)
      Candidate c;
      c.members = P.list();
      c.output = sink;
      c.n_dense = nd;
      std::vector<int> ins;
      std::vector<int> gins;
      for (int v : c.members) {
        for (auto& r : g.prims[v].in) {
          if (r.is_input) gins.push_back(r.id);
          else if (!P.test(r.id)) ins.push_back(r.id);
        }
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
  std::sort(out.begin(), out.end(), [](const Candidate& x, const Candidate& y) {
    if (x.output != y.output) return x.output < y.output;
    if (x.members.size() != y.members.size()) return x.members.size() < y.members.size();
    return x.members < y.members;
  });
  return out;
}

}  // namespace korch
