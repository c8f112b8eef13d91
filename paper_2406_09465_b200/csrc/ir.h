// Primitive-graph IR G=(P,E) and operator fission.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "json.h"

namespace korch {

enum class DType : int { F32 = 0, BF16 = 1 };
inline int dtype_size(DType t) { return t == DType::F32 ? 4 : 2; }
inline const char* dtype_name(DType t) { return t == DType::F32 ? "f32" : "bf16"; }

// The four primitive categories of P:157-192 (Table 1).
enum class Kind : int {
  // elementwise, unary
  Exp, Sqrt, Erf, Relu, Sigmoid, Tanh, Neg, HardSwish, Softplus, Identity,
  // elementwise, scalar constant
  AddC, MulC, DivC,
  // elementwise, binary
  Add, Sub, Mul, Div,
  // reduce and broadcast
  Reduce, Broadcast, MaxPool,
  // layout transformation
  Transpose, Reshape, Slice, Pad, Concat,
  // linear transformation
  MatMul, Conv2d,
  // constant tensor (R1's ones C_s)
  Constant,
};

enum class RedOp : int { Sum = 0, Mean = 1, Max = 2 };

const char* kind_name(Kind k);
bool kind_from_name(const std::string& s, Kind* k);
bool is_unary(Kind k);
bool is_scalar_op(Kind k);
bool is_binary(Kind k);
bool is_elementwise(Kind k);
bool is_layout(Kind k);

using Shape = std::vector<int64_t>;
inline int64_t numel(const Shape& s) {
  int64_t n = 1;
  for (auto d : s) n *= d;
  return n;
}

struct Ref {
  bool is_input = false;  // true: graph input index; false: primitive id
  int id = -1;
};

struct Prim {
  int id = -1;
  Kind kind = Kind::Identity;
  std::vector<Ref> in;
  Shape shape;
  DType dtype = DType::F32;  // storage dtype when materialised
  // attributes
  double c = 0;                 // AddC/MulC/DivC constant, Constant value, Pad value
  int axis = 0;                 // Reduce / Broadcast / Slice / Concat axis
  RedOp red = RedOp::Sum;       // Reduce aggregator
  int64_t size = 0;             // Broadcast extent
  std::vector<int> perm;        // Transpose
  Shape new_shape;              // Reshape / Constant
  int64_t start = 0, end = 0;   // Slice
  std::vector<std::pair<int64_t, int64_t>> pads;  // Pad: per-axis (low, high)
  bool reflect = false;         // Pad mode
  int stride[2] = {1, 1}, cpad[2] = {0, 0}, groups = 1;  // Conv2d
  int pk = 0, pstride = 1, ppad = 0;                     // MaxPool
  // port broadcast of graph-input operands (reading A13): for input slot s,
  // port_axes[s] maps each input axis to an output axis; empty = right-aligned.
  std::vector<std::vector<int>> port_axes;
  int op_id = -1;  // operator this primitive came from (operator-aligned baseline)
};

struct InputSpec {
  std::string name;
  Shape shape;
  DType dtype = DType::F32;
};

struct Graph {
  DType dtype = DType::F32;  // storage dtype of computed tensors (A20/A25)
  std::vector<InputSpec> inputs;
  std::vector<Prim> prims;
  std::vector<int> outputs;  // T
  // derived
  std::vector<std::vector<int>> preds, succs;  // primitive edges only
  std::vector<int> topo;                       // Kahn, smallest id first
  std::vector<int> topo_index;

  const Shape& shape_of(const Ref& r) const {
    return r.is_input ? inputs[r.id].shape : prims[r.id].shape;
  }
  DType dtype_of(const Ref& r) const {
    return r.is_input ? inputs[r.id].dtype : prims[r.id].dtype;
  }
  bool is_dense_linear(int p) const;  // reading A18
  void finalize();                    // preds/succs/topo; throws on cycle
};

struct KorchError : std::runtime_error {
  int code;
  KorchError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Parse operator- or primitive-level JSON; operator level runs fission.
Graph load_graph(const char* json, size_t n);
std::string dump_graph(const Graph& g);
std::string validate_graph(const Graph& g);
Shape infer_shape(const Graph& g, const Prim& p);
// R1-R3 at every Softmax -> MatMul site (rewrites.cpp); renumbers primitives.
void apply_r1_r3(Graph& g);

}  // namespace korch
