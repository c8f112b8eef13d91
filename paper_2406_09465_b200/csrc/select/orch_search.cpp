// Exact kernel-orchestration solver (include/korch_select.h): A* over producer
// assignments.  Host-side, caller-side code; not linked into
// libkorch.so.
//
// Search space.  A selection is optimal only if every materialised tensor has exactly
// one producer (A7: costs are positive, so a second producer can be dropped without
// breaking Eq. 3/4).  Resolve the materialised tensors from the LAST (in topological
// order) to the first: the pending set S holds the tensors that must still get a
// producer.  Expanding S picks t = max(S) and, for every candidate p with output t,
// moves to S' = (S \ {t}) u I(p).  Every input of p precedes t, and every tensor
// resolved before t comes after it, so nothing in I(p) has been resolved yet and the
// cost-to-go depends on S alone: the search graph is a DAG over pending sets and the
// optimal orchestration is a shortest path from T to the empty set (edge weight
// (c_p, 1): cost first, kernel count second -- reading A8).
//
// Heuristic.  h(S) = (sum_{t in S} min_p c_p, |S|): distinct pending tensors need
// distinct kernels (one output per kernel), so h never overestimates.  It is also
// consistent: h(S) <= (c_p, 1) + h(S') because S \ {t} is a subset of S'.  Hence the
// first time the empty set is popped its path is optimal (lexicographically in
// (cost, kernels)).  A greedy dive gives an incumbent for pruning.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <queue>
#include <unordered_map>
#include <vector>

#include "../../../include/korch_select.h"

namespace {

template <int W>
struct Bits {
  uint64_t w[W];
  bool operator==(const Bits& o) const { return std::memcmp(w, o.w, sizeof w) == 0; }
  bool empty() const {
    for (int i = 0; i < W; ++i)
      if (w[i]) return false;
    return true;
  }
  int top() const {  // highest set bit (S non-empty)
    for (int i = W - 1; i >= 0; --i)
      if (w[i]) return i * 64 + 63 - __builtin_clzll(w[i]);
    return -1;
  }
  bool has(int b) const { return (w[b >> 6] >> (b & 63)) & 1; }
  void set(int b) { w[b >> 6] |= 1ull << (b & 63); }
  void clr(int b) { w[b >> 6] &= ~(1ull << (b & 63)); }
};

template <int W>
struct BitsHash {
  size_t operator()(const Bits<W>& b) const {
    uint64_t h = 1469598103934665603ull;
    for (int i = 0; i < W; ++i) {
      h ^= b.w[i] + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
      h *= 1099511628211ull;
    }
    return (size_t)h;
  }
};

struct Key {  // (cost, kernels), compared lexicographically
  int64_t c;
  int64_t k;
  bool operator<(const Key& o) const { return c != o.c ? c < o.c : k < o.k; }
  bool operator<=(const Key& o) const { return !(o < *this); }
  Key operator+(const Key& o) const { return {c + o.c, k + o.k}; }
};

struct Problem {
  int n = 0, m = 0;
  const int32_t* out = nullptr;
  const int32_t* off = nullptr;
  const int32_t* in = nullptr;
  const int64_t* cost = nullptr;
  std::vector<std::vector<int32_t>> producers;  // tensor -> candidates, cheapest first
  std::vector<int64_t> minc;                    // tensor -> cheapest producer (or -1)
};

template <int W>
int32_t solve(const Problem& P, const std::vector<int32_t>& req, int64_t max_states, double tlim, int64_t* best_cost,
              int32_t* sel, int64_t* n_expanded) {
  using B = Bits<W>;
  auto t0 = std::chrono::steady_clock::now();
  auto h_of = [&](const B& s) {
    Key h{0, 0};
    for (int i = 0; i < W; ++i) {
      uint64_t x = s.w[i];
      while (x) {
        int b = i * 64 + __builtin_ctzll(x);
        x &= x - 1;
        h.c += P.minc[b];
        h.k += 1;
      }
    }
    return h;
  };
  auto next_state = [&](const B& s, int t, int p) {
    B n = s;
    n.clr(t);
    for (int32_t e = P.off[p]; e < P.off[p + 1]; ++e) n.set(P.in[e]);
    return n;
  };

  B start{};
  for (int32_t t : req) start.set(t);
  for (int32_t t : req)
    if (P.producers[t].empty()) return KORCH_SEL_E_INFEASIBLE;

  // incumbent: greedy dive (cheapest producer of the latest pending tensor); pending
  // tensors without a producer make the dive fail, which only costs the bound
  Key ub{INT64_MAX, INT64_MAX};
  {
    B s = start;
    Key g{0, 0};
    bool ok = true;
    while (!s.empty()) {
      int t = s.top();
      if (P.producers[t].empty()) { ok = false; break; }
      int p = P.producers[t][0];
      g = g + Key{P.cost[p], 1};
      s = next_state(s, t, p);
    }
    if (ok) ub = g;
  }

  struct Node {
    B s;
    Key g;
    int32_t parent;
    int32_t cand;
  };
  std::vector<Node> nodes;
  nodes.reserve(1 << 16);
  std::unordered_map<B, Key, BitsHash<W>> best;
  best.reserve(1 << 16);
  struct QE {
    Key f;
    int32_t idx;
  };
  auto cmp = [](const QE& a, const QE& b) { return b.f < a.f; };  // min-heap on f
  std::priority_queue<QE, std::vector<QE>, decltype(cmp)> open(cmp);

  nodes.push_back({start, {0, 0}, -1, -1});
  best[start] = {0, 0};
  open.push({h_of(start), 0});
  int64_t expanded = 0;
  int32_t goal = -1;
  while (!open.empty()) {
    QE q = open.top();
    open.pop();
    const Node cur = nodes[q.idx];
    auto it = best.find(cur.s);
    if (it != best.end() && it->second < cur.g) continue;  // stale entry
    if (cur.s.empty()) { goal = q.idx; break; }
    if (++expanded > max_states || (int64_t)nodes.size() > 4 * max_states) break;
    if (tlim > 0 && (expanded & 1023) == 0 &&
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > tlim)
      break;
    int t = cur.s.top();
    Key hs = h_of(cur.s);
    for (int32_t p : P.producers[t]) {
      B ns = next_state(cur.s, t, p);
      bool dead = false;  // a pending tensor nobody produces: no completion
      Key hn{0, 0};
      for (int i = 0; i < W && !dead; ++i) {
        uint64_t x = ns.w[i];
        while (x) {
          int b = i * 64 + __builtin_ctzll(x);
          x &= x - 1;
          if (P.minc[b] < 0) { dead = true; break; }
          hn.c += P.minc[b];
          hn.k += 1;
        }
      }
      if (dead) continue;
      Key g = cur.g + Key{P.cost[p], 1};
      Key f = g + hn;
      if (ub < f) continue;
      auto bi = best.find(ns);
      if (bi != best.end() && bi->second <= g) continue;
      best[ns] = g;
      nodes.push_back({ns, g, q.idx, p});
      open.push({f, (int32_t)nodes.size() - 1});
    }
    (void)hs;
  }
  if (n_expanded) *n_expanded = expanded;
  if (goal < 0) return open.empty() ? KORCH_SEL_E_INFEASIBLE : KORCH_SEL_E_LIMIT;
  std::fill(sel, sel + P.m, 0);
  int64_t tot = 0;
  for (int32_t i = goal; nodes[i].parent >= 0; i = nodes[i].parent) {
    sel[nodes[i].cand] = 1;
    tot += P.cost[nodes[i].cand];
  }
  *best_cost = tot;
  return KORCH_SEL_OK;
}

}  // namespace

extern "C" int32_t korch_select_exact(int32_t n_tensors, int32_t n_cands, const int32_t* cand_output,
                                      const int32_t* cand_in_off, const int32_t* cand_in, const int64_t* cand_cost,
                                      int32_t n_required, const int32_t* required, int64_t max_states,
                                      double time_limit_s, int64_t* best_cost, int32_t* sel, int64_t* n_expanded) {
  if (n_tensors <= 0 || n_tensors > 512 || n_cands < 0 || n_required < 0 || !best_cost || (n_cands > 0 && !sel) ||
      (n_cands > 0 && (!cand_output || !cand_in_off || !cand_cost)) || (n_required > 0 && !required))
    return KORCH_SEL_E_ARG;
  Problem P;
  P.n = n_tensors;
  P.m = n_cands;
  P.out = cand_output;
  P.off = cand_in_off;
  P.in = cand_in;
  P.cost = cand_cost;
  P.producers.assign(n_tensors, {});
  P.minc.assign(n_tensors, -1);
  for (int32_t i = 0; i < n_cands; ++i) {
    int32_t o = cand_output[i];
    if (o < 0 || o >= n_tensors || cand_cost[i] < 1 || cand_cost[i] >= (int64_t)1 << 40) return KORCH_SEL_E_ARG;
    for (int32_t e = cand_in_off[i]; e < cand_in_off[i + 1]; ++e)
      if (cand_in[e] < 0 || cand_in[e] >= o) return KORCH_SEL_E_ARG;  // inputs precede the output
    P.producers[o].push_back(i);
  }
  for (int t = 0; t < n_tensors; ++t) {
    auto& ps = P.producers[t];
    std::sort(ps.begin(), ps.end(), [&](int32_t a, int32_t b) {
      return cand_cost[a] != cand_cost[b] ? cand_cost[a] < cand_cost[b] : a < b;
    });
    if (!ps.empty()) P.minc[t] = cand_cost[ps[0]];
  }
  std::vector<int32_t> req(required, required + n_required);
  for (int32_t t : req)
    if (t < 0 || t >= n_tensors) return KORCH_SEL_E_ARG;
  if (max_states <= 0) max_states = 50000000;
  if (n_expanded) *n_expanded = 0;
  if (req.empty()) {
    std::fill(sel, sel + n_cands, 0);
    *best_cost = 0;
    return KORCH_SEL_OK;
  }
  int w = (n_tensors + 63) / 64;
  if (w <= 1) return solve<1>(P, req, max_states, time_limit_s, best_cost, sel, n_expanded);
  if (w <= 2) return solve<2>(P, req, max_states, time_limit_s, best_cost, sel, n_expanded);
  if (w <= 4) return solve<4>(P, req, max_states, time_limit_s, best_cost, sel, n_expanded);
  return solve<8>(P, req, max_states, time_limit_s, best_cost, sel, n_expanded);
}
