// Kernel identifier: Alg. 1 over execution states.
#pragma once
#include <cstdint>
#include <cstring>
#include <functional>
#include <vector>

#include "ir.h"

namespace korch {

constexpr int kMaxPrims = 256;  // one partition (H4) holds at most this many primitives

struct Bits {
  uint64_t w[kMaxPrims / 64] = {0, 0, 0, 0};
  void set(int i) { w[i >> 6] |= 1ull << (i & 63); }
  void reset(int i) { w[i >> 6] &= ~(1ull << (i & 63)); }
  bool test(int i) const { return (w[i >> 6] >> (i & 63)) & 1; }
  int count() const {
    int c = 0;
    for (auto x : w) c += __builtin_popcountll(x);
    return c;
  }
  bool operator==(const Bits& o) const { return std::memcmp(w, o.w, sizeof(w)) == 0; }
  // strict subset
  bool subset_of(const Bits& o) const {
    bool eq = true;
    for (int i = 0; i < kMaxPrims / 64; ++i) {
      if (w[i] & ~o.w[i]) return false;
      if (w[i] != o.w[i]) eq = false;
    }
    return !eq;
  }
  Bits minus(const Bits& o) const {
    Bits r;
    for (int i = 0; i < kMaxPrims / 64; ++i) r.w[i] = w[i] & ~o.w[i];
    return r;
  }
  std::vector<int> list() const {
    std::vector<int> r;
    for (int i = 0; i < kMaxPrims; ++i)
      if (test(i)) r.push_back(i);
    return r;
  }
};

struct BitsHash {
  size_t operator()(const Bits& b) const {
    uint64_t h = 1469598103934665603ull;
    for (auto x : b.w) { h ^= x; h *= 1099511628211ull; h ^= h >> 29; }
    return (size_t)h;
  }
};

struct Candidate {
  std::vector<int> members;       // P', ascending
  int output = -1;                // o (unique sink, reading A4)
  std::vector<int> extra_outputs; // E: secondary materialised outputs (N1, reading A32), ascending
  std::vector<int> inputs;        // primitive inputs (I row)
  std::vector<int> graph_inputs;  // graph-input indices read
  int klass = 0;                  // KORCH_CLASS_*
  int n_dense = 0;
  int64_t bytes = 0;
  double flops = 0;
  std::string signature;
  std::string reject_reason;
  int part = 0;                   // partition part (A17)
};

struct EnumOpts {
  int max_prims = 16;
  bool keep_multi_linear = false;
  int64_t max_states = 1000000;
  int partition_max = 0;          // > 0: partition into parts of about this many primitives
  bool attention_pairs = false;   // N2: keep MatMul pairs where the first feeds the second's A
  int max_outputs = 1;            // N1: > 1 adds (P', o, E) with |E| <= max_outputs - 1 (reading A32)
};

// Reading A17: parts of the topological order separated at articulation tensors.
std::vector<std::vector<int>> partition_graph(const Graph& g, int max_nodes);

// Runs Alg. 1 (per partition part) with B seeded with the empty state (reading A1);
// returns the unique-sink, pruned candidates in canonical order and the state count.
std::vector<Candidate> enumerate_candidates(const Graph& g, const EnumOpts& o, int64_t* n_states,
                                            std::vector<std::vector<int>>* parts = nullptr);

}  // namespace korch
