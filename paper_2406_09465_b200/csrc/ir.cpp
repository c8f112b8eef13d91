// Primitive-graph IR, shape inference, JSON I/O and operator fission.
//
// Fission rules (readings A9-A16).
// Primitive ids: operators in Kahn order (smallest id first), then each
// rule's primitives in the listed order.
#include "ir.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <queue>
#include <sstream>

#include "../../include/korch.h"

namespace korch {

static const char* kKindNames[] = {
    "exp", "sqrt", "erf", "relu", "sigmoid", "tanh", "neg", "hardswish", "softplus", "identity",
    "addc", "mulc", "divc", "add", "sub", "mul", "div", "reduce", "broadcast", "maxpool",
    "transpose", "reshape", "slice", "pad", "concat", "matmul", "conv2d", "constant"};

const char* kind_name(Kind k) { return kKindNames[(int)k]; }
bool kind_from_name(const std::string& s, Kind* k) {
  for (int i = 0; i <= (int)Kind::Constant; ++i)
    if (s == kKindNames[i]) { *k = (Kind)i; return true; }
  return false;
}
bool is_unary(Kind k) { return (int)k <= (int)Kind::Identity; }
bool is_scalar_op(Kind k) { return k == Kind::AddC || k == Kind::MulC || k == Kind::DivC; }
bool is_binary(Kind k) { return k == Kind::Add || k == Kind::Sub || k == Kind::Mul || k == Kind::Div; }
bool is_elementwise(Kind k) { return is_unary(k) || is_scalar_op(k) || is_binary(k); }
bool is_layout(Kind k) {
  return k == Kind::Transpose || k == Kind::Reshape || k == Kind::Slice || k == Kind::Pad ||
         k == Kind::Concat;
}

bool Graph::is_dense_linear(int p) const {
  const Prim& q = prims[p];
  if (q.kind == Kind::MatMul) return true;
  if (q.kind == Kind::Conv2d) return shape_of(q.in[1])[1] >= 16;  // channels per group (A18)
  return false;
}

void Graph::finalize() {
  int n = (int)prims.size();
  preds.assign(n, {});
  succs.assign(n, {});
  for (auto& p : prims)
    for (auto& r : p.in)
      if (!r.is_input) {
        if (r.id < 0 || r.id >= n) throw KorchError(KORCH_E_PARSE, "dangling primitive reference");
        if (std::find(preds[p.id].begin(), preds[p.id].end(), r.id) == preds[p.id].end())
          preds[p.id].push_back(r.id);
      }
  for (int v = 0; v < n; ++v) {
    std::sort(preds[v].begin(), preds[v].end());
    for (int u : preds[v]) succs[u].push_back(v);
  }
  std::vector<int> indeg(n);
  std::priority_queue<int, std::vector<int>, std::greater<int>> pq;
  for (int v = 0; v < n; ++v) {
    indeg[v] = (int)preds[v].size();
    if (!indeg[v]) pq.push(v);
  }
  topo.clear();
  while (!pq.empty()) {
    int v = pq.top();
    pq.pop();
    topo.push_back(v);
    for (int w : succs[v])
      if (--indeg[w] == 0) pq.push(w);
  }
  if ((int)topo.size() != n) throw KorchError(KORCH_E_CYCLE, "primitive graph has a cycle");
  topo_index.assign(n, 0);
  for (int i = 0; i < n; ++i) topo_index[topo[i]] = i;
}

// ---------------------------------------------------------------- shapes
[[noreturn]] static void shape_fail(const Prim& p, const std::string& m) {
  throw KorchError(KORCH_E_SHAPE, std::string("shape error at primitive ") + std::to_string(p.id) +
                                      " (" + kind_name(p.kind) + "): " + m);
}

Shape infer_shape(const Graph& g, const Prim& p) {
  auto in = [&](int i) -> const Shape& {
    if (i >= (int)p.in.size()) shape_fail(p, "missing input");
    return g.shape_of(p.in[i]);
  };
  Kind k = p.kind;
  if (is_unary(k) || is_scalar_op(k)) return in(0);
  if (is_binary(k)) {
    const Shape &a = in(0), &b = in(1);
    if (a == b) return a;
    // port broadcast: the graph-input operand is broadcast onto the other
    int port = p.in[1].is_input ? 1 : (p.in[0].is_input ? 0 : -1);
    if (port < 0) shape_fail(p, "computed operands of different shapes need explicit broadcasts");
    const Shape& full = port == 1 ? a : b;
    const Shape& part = port == 1 ? b : a;
    std::vector<int> axes;
    if ((int)p.port_axes.size() > port && !p.port_axes[port].empty()) axes = p.port_axes[port];
    else {
      if (part.size() > full.size()) shape_fail(p, "port operand has higher rank");
      for (size_t i = 0; i < part.size(); ++i) axes.push_back((int)(full.size() - part.size() + i));
    }
    if (axes.size() != part.size()) shape_fail(p, "port_axes rank mismatch");
    for (size_t i = 0; i < part.size(); ++i) {
      if (axes[i] < 0 || axes[i] >= (int)full.size()) shape_fail(p, "port axis out of range");
      if (part[i] != 1 && part[i] != full[axes[i]]) shape_fail(p, "port extent mismatch");
    }
    return full;
  }
  switch (k) {
    case Kind::Reduce: {
      Shape s = in(0);
      if (p.axis < 0 || p.axis >= (int)s.size()) shape_fail(p, "reduce axis");
      s.erase(s.begin() + p.axis);
      return s;
    }
    case Kind::Broadcast: {
      Shape s = in(0);
      if (p.axis < 0 || p.axis > (int)s.size()) shape_fail(p, "broadcast axis");
      s.insert(s.begin() + p.axis, p.size);
      return s;
    }
    case Kind::Transpose: {
      const Shape& s = in(0);
      if (p.perm.size() != s.size()) shape_fail(p, "perm rank");
      Shape r;
      for (int a : p.perm) r.push_back(s.at(a));
      return r;
    }
    case Kind::Reshape:
      if (numel(p.new_shape) != numel(in(0))) shape_fail(p, "reshape element count");
      return p.new_shape;
    case Kind::Slice: {
      Shape s = in(0);
      if (p.axis < 0 || p.axis >= (int)s.size() || p.start < 0 || p.end > s[p.axis] || p.start >= p.end)
        shape_fail(p, "slice range");
      s[p.axis] = p.end - p.start;
      return s;
    }
    case Kind::Pad: {
      Shape s = in(0);
      if (p.pads.size() != s.size()) shape_fail(p, "pads rank");
      for (size_t i = 0; i < s.size(); ++i) s[i] += p.pads[i].first + p.pads[i].second;
      return s;
    }
    case Kind::Concat: {
      Shape s = in(0);
      int64_t t = 0;
      for (size_t i = 0; i < p.in.size(); ++i) t += in((int)i).at(p.axis);
      s[p.axis] = t;
      return s;
    }
    case Kind::MatMul: {
      const Shape &a = in(0), &b = in(1);
      if (a.size() < 2 || b.size() < 2) shape_fail(p, "matmul rank");
      if (a[a.size() - 1] != b[b.size() - 2]) shape_fail(p, "contraction mismatch");
      Shape ba(a.begin(), a.end() - 2), bb(b.begin(), b.end() - 2);
      Shape batch;
      if (bb.empty()) batch = ba;
      else if (ba == bb) batch = ba;
      else shape_fail(p, "batch dims differ");
      batch.push_back(a[a.size() - 2]);
      batch.push_back(b.back());
      return batch;
    }
    case Kind::Conv2d: {
      const Shape &x = in(0), &w = in(1);
      if (x.size() != 4 || w.size() != 4 || x[1] != w[1] * p.groups) shape_fail(p, "conv shapes");
      return {x[0], w[0], (x[2] + 2 * p.cpad[0] - w[2]) / p.stride[0] + 1,
              (x[3] + 2 * p.cpad[1] - w[3]) / p.stride[1] + 1};
    }
    case Kind::MaxPool: {
      const Shape& x = in(0);
      return {x[0], x[1], (x[2] + 2 * p.ppad - p.pk) / p.pstride + 1,
              (x[3] + 2 * p.ppad - p.pk) / p.pstride + 1};
    }
    case Kind::Constant:
      return p.new_shape;
    default:
      shape_fail(p, "unknown kind");
  }
}

// ---------------------------------------------------------------- JSON helpers
static DType parse_dtype(const std::string& s) {
  if (s == "f32") return DType::F32;
  if (s == "bf16") return DType::BF16;
  throw KorchError(KORCH_E_PARSE, "unknown dtype '" + s + "'");
}

static void read_prim_attrs(Prim& p, const Json& a) {
  auto num = [&](const char* k, double d) { return a.has(k) ? a[k].as_num() : d; };
  auto integ = [&](const char* k, int64_t d) { return a.has(k) ? a[k].as_int() : d; };
  switch (p.kind) {
    case Kind::AddC: case Kind::MulC: case Kind::DivC: p.c = a["c"].as_num(); break;
    case Kind::Reduce: {
      p.axis = (int)a["axis"].as_int();
      std::string op = a.has("op") ? a["op"].as_str() : "sum";
      p.red = op == "sum" ? RedOp::Sum : op == "mean" ? RedOp::Mean : op == "max" ? RedOp::Max
                                                                                    : throw KorchError(KORCH_E_PARSE, "reduce op");
      break;
    }
    case Kind::Broadcast: p.axis = (int)a["axis"].as_int(); p.size = a["size"].as_int(); break;
    case Kind::Transpose: for (auto v : a["perm"].as_ints()) p.perm.push_back((int)v); break;
    case Kind::Reshape: p.new_shape = a["shape"].as_ints(); break;
    case Kind::Slice:
      p.axis = (int)a["axis"].as_int(); p.start = a["start"].as_int(); p.end = a["end"].as_int(); break;
    case Kind::Pad:
      for (auto& pr : a["pads"].arr) p.pads.push_back({pr.at(0).as_int(), pr.at(1).as_int()});
      p.reflect = a.has("mode") && a["mode"].as_str() == "reflect";
      p.c = num("value", 0.0);
      break;
    case Kind::Concat: p.axis = (int)a["axis"].as_int(); break;
    case Kind::Conv2d: {
      if (a.has("stride")) { auto s = a["stride"].as_ints(); p.stride[0] = (int)s[0]; p.stride[1] = (int)s[1]; }
      if (a.has("pads")) { auto s = a["pads"].as_ints(); p.cpad[0] = (int)s[0]; p.cpad[1] = (int)s[1]; }
      p.groups = (int)integ("groups", 1);
      break;
    }
    case Kind::MaxPool:
      p.pk = (int)a["k"].as_int(); p.pstride = (int)a["stride"].as_int(); p.ppad = (int)integ("pad", 0); break;
    case Kind::Constant: p.new_shape = a["shape"].as_ints(); p.c = a["value"].as_num(); break;
    default: break;
  }
  if (a.has("port_axes")) {
    for (auto& kv : a["port_axes"].obj) {
      int slot = std::stoi(kv.first);
      if ((int)p.port_axes.size() <= slot) p.port_axes.resize(slot + 1);
      for (auto v : kv.second.as_ints()) p.port_axes[slot].push_back((int)v);
    }
  }
}

// ---------------------------------------------------------------- fission
namespace {
struct Builder {
  Graph& g;
  int op_id = -1;
  explicit Builder(Graph& gg) : g(gg) {}
  Ref add(Prim p, std::vector<Ref> in) {
    p.id = (int)g.prims.size();
    p.in = std::move(in);
    p.dtype = g.dtype;
    p.op_id = op_id;
    p.shape = infer_shape(g, p);
    g.prims.push_back(p);
    return Ref{false, p.id};
  }
  Ref unary(Kind k, Ref x, double c = 0) {
    Prim p; p.kind = k; p.c = c;
    return add(p, {x});
  }
  Ref binary(Kind k, Ref a, Ref b, int port_slot = -1, std::vector<int> axes = {}) {
    Prim p; p.kind = k;
    if (port_slot >= 0) { p.port_axes.resize(port_slot + 1); p.port_axes[port_slot] = axes; }
    return add(p, {a, b});
  }
  Ref reduce(Ref x, int axis, RedOp op) { Prim p; p.kind = Kind::Reduce; p.axis = axis; p.red = op; return add(p, {x}); }
  Ref bcast(Ref x, int axis, int64_t size) { Prim p; p.kind = Kind::Broadcast; p.axis = axis; p.size = size; return add(p, {x}); }
  Ref reshape(Ref x, Shape s) { Prim p; p.kind = Kind::Reshape; p.new_shape = s; return add(p, {x}); }
};

// LayerNorm's first nine primitives over `axis` (reading A10).
Ref ln_core(Builder& b, Ref x, int axis, double eps) {
  int64_t n = b.g.shape_of(x)[axis];
  Ref m = b.reduce(x, axis, RedOp::Mean);
  Ref bm = b.bcast(m, axis, n);
  Ref c = b.binary(Kind::Sub, x, bm);
  Ref s = b.binary(Kind::Mul, c, c);
  Ref v = b.reduce(s, axis, RedOp::Mean);
  Ref ve = b.unary(Kind::AddC, v, eps);
  Ref sd = b.unary(Kind::Sqrt, ve);
  Ref bsd = b.bcast(sd, axis, n);
  return b.binary(Kind::Div, c, bsd);
}

Ref elementwise_binary(Builder& b, Kind k, Ref x, Ref y) {
  const Shape sx = b.g.shape_of(x), sy = b.g.shape_of(y);
  if (sx == sy) return b.binary(k, x, y);
  if (y.is_input && sy.size() <= sx.size()) return b.binary(k, x, y);  // port broadcast (A13)
  if (x.is_input && sx.size() <= sy.size()) return b.binary(k, x, y);
  if (sx.size() < sy.size()) {
    for (size_t i = 0; i < sy.size() - sx.size(); ++i) x = b.bcast(x, 0, sy[sy.size() - sx.size() - 1 - i]);
    return b.binary(k, x, y);
  }
  if (sy.size() < sx.size()) {
    for (size_t i = 0; i < sx.size() - sy.size(); ++i) y = b.bcast(y, 0, sx[sx.size() - sy.size() - 1 - i]);
    return b.binary(k, x, y);
  }
  throw KorchError(KORCH_E_UNSUPPORTED, "unsupported broadcast between computed tensors");
}

int norm_axis(int64_t a, size_t rank) { return (int)(a < 0 ? a + (int64_t)rank : a); }

Graph fission_graph(const Json& j) {
  Graph g;
  g.dtype = parse_dtype(j["dtype"].as_str());
  std::map<std::string, int> in_idx;
  for (auto& s : j["inputs"].arr) {
    InputSpec is;
    is.name = s["name"].as_str();
    is.shape = s["shape"].as_ints();
    is.dtype = s.has("dtype") ? parse_dtype(s["dtype"].as_str()) : g.dtype;
    in_idx[is.name] = (int)g.inputs.size();
    g.inputs.push_back(is);
  }
  // operator DAG in Kahn order, smallest id first
  const auto& nodes = j["nodes"].arr;
  std::map<int64_t, const Json*> ops;
  for (auto& n : nodes) ops[n["id"].as_int()] = &n;
  std::map<int64_t, std::vector<int64_t>> users;
  std::map<int64_t, int> indeg;
  for (auto& kv : ops) {
    indeg[kv.first] = 0;
    std::vector<int64_t> deps;
    for (auto& r : (*kv.second)["inputs"].arr)
      if (r.has("node")) {
        int64_t d = r["node"].as_int();
        if (!ops.count(d)) throw KorchError(KORCH_E_PARSE, "unknown node reference");
        if (std::find(deps.begin(), deps.end(), d) == deps.end()) deps.push_back(d);
      }
    indeg[kv.first] = (int)deps.size();
    for (auto d : deps) users[d].push_back(kv.first);
  }
  std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> pq;
  for (auto& kv : indeg) if (!kv.second) pq.push(kv.first);
  std::vector<int64_t> order;
  while (!pq.empty()) {
    int64_t v = pq.top(); pq.pop();
    order.push_back(v);
    for (auto u : users[v]) if (--indeg[u] == 0) pq.push(u);
  }
  if (order.size() != ops.size()) throw KorchError(KORCH_E_CYCLE, "operator graph has a cycle");

  Builder b(g);
  std::map<int64_t, int> out_of;
  static const std::map<std::string, Kind> simple = {
      {"Exp", Kind::Exp}, {"Sqrt", Kind::Sqrt}, {"Erf", Kind::Erf}, {"Relu", Kind::Relu},
      {"Sigmoid", Kind::Sigmoid}, {"Tanh", Kind::Tanh}, {"Neg", Kind::Neg},
      {"HardSwish", Kind::HardSwish}, {"Softplus", Kind::Softplus}, {"Identity", Kind::Identity},
      {"AddC", Kind::AddC}, {"MulC", Kind::MulC}, {"DivC", Kind::DivC},
      {"Transpose", Kind::Transpose}, {"Reshape", Kind::Reshape}, {"Slice", Kind::Slice},
      {"Pad", Kind::Pad}, {"Concat", Kind::Concat}, {"MaxPool", Kind::MaxPool}, {"Broadcast", Kind::Broadcast}};
  static const std::map<std::string, Kind> bins = {
      {"Add", Kind::Add}, {"Sub", Kind::Sub}, {"Mul", Kind::Mul}, {"Div", Kind::Div}};
  static const std::map<std::string, RedOp> reds = {
      {"ReduceSum", RedOp::Sum}, {"ReduceMean", RedOp::Mean}, {"ReduceMax", RedOp::Max}};

  for (int64_t oid : order) {
    const Json& op = *ops[oid];
    b.op_id = (int)oid;
    std::vector<Ref> ins;
    for (auto& r : op["inputs"].arr) {
      if (r.has("node")) ins.push_back(Ref{false, out_of.at(r["node"].as_int())});
      else {
        auto it = in_idx.find(r["input"].as_str());
        if (it == in_idx.end()) throw KorchError(KORCH_E_PARSE, "unknown graph input '" + r["input"].as_str() + "'");
        ins.push_back(Ref{true, it->second});
      }
    }
    const std::string& k = op["kind"].as_str();
    const Json& at = op["attrs"];
    auto need = [&](size_t n) { if (ins.size() < n) throw KorchError(KORCH_E_PARSE, k + ": too few inputs"); };
    Ref res;
    if (simple.count(k)) {
      need(1);
      Prim p; p.kind = simple.at(k);
      read_prim_attrs(p, at);
      if (p.kind == Kind::Transpose || p.kind == Kind::Slice || p.kind == Kind::Concat) {}
      res = b.add(p, ins);
    } else if (bins.count(k)) {
      need(2);
      res = elementwise_binary(b, bins.at(k), ins[0], ins[1]);
    } else if (reds.count(k)) {
      need(1);
      res = b.reduce(ins[0], norm_axis(at["axis"].as_int(), g.shape_of(ins[0]).size()), reds.at(k));
    } else if (k == "Softmax") {  // Fig. 5
      need(1);
      int ax = norm_axis(at["axis"].as_int(), g.shape_of(ins[0]).size());
      Ref e = b.unary(Kind::Exp, ins[0]);
      Ref r = b.reduce(e, ax, RedOp::Sum);
      Ref bc = b.bcast(r, ax, g.shape_of(ins[0])[ax]);
      res = b.binary(Kind::Div, e, bc);
    } else if (k == "LayerNorm") {  // A10
      need(1);
      int rank = (int)g.shape_of(ins[0]).size();
      int ax = norm_axis(at.has("axis") ? at["axis"].as_int() : -1, rank);
      if (ax != rank - 1) throw KorchError(KORCH_E_UNSUPPORTED, "LayerNorm over a non-last axis");
      double eps = at.has("eps") ? at["eps"].as_num() : 1e-5;
      res = ln_core(b, ins[0], ax, eps);
      if (ins.size() > 1) res = b.binary(Kind::Mul, res, ins[1]);
      if (ins.size() > 2) res = b.binary(Kind::Add, res, ins[2]);
    } else if (k == "InstanceNorm") {  // A11
      need(3);
      Shape s = g.shape_of(ins[0]);
      if (s.size() != 4) throw KorchError(KORCH_E_SHAPE, "InstanceNorm expects NCHW");
      Ref r = b.reshape(ins[0], {s[0], s[1], s[2] * s[3]});
      Ref y = ln_core(b, r, 2, at.has("eps") ? at["eps"].as_num() : 1e-5);
      y = b.binary(Kind::Mul, y, ins[1], 1, {1});
      y = b.binary(Kind::Add, y, ins[2], 1, {1});
      res = b.reshape(y, s);
    } else if (k == "GELU") {  // A12
      need(1);
      Ref a = b.unary(Kind::DivC, ins[0], std::sqrt(2.0));
      Ref e = b.unary(Kind::Erf, a);
      Ref f = b.unary(Kind::AddC, e, 1.0);
      Ref m = b.binary(Kind::Mul, ins[0], f);
      res = b.unary(Kind::MulC, m, 0.5);
    } else if (k == "SiLU") {
      need(1);
      Ref s = b.unary(Kind::Sigmoid, ins[0]);
      res = b.binary(Kind::Mul, ins[0], s);
    } else if (k == "Mish") {
      need(1);
      Ref s = b.unary(Kind::Softplus, ins[0]);
      Ref t = b.unary(Kind::Tanh, s);
      res = b.binary(Kind::Mul, ins[0], t);
    } else if (k == "MatMul") {
      need(2);
      Prim p; p.kind = Kind::MatMul;
      res = b.add(p, {ins[0], ins[1]});
    } else if (k == "Conv") {
      need(2);
      Prim p; p.kind = Kind::Conv2d;
      read_prim_attrs(p, at);
      res = b.add(p, {ins[0], ins[1]});
      if (ins.size() > 2) res = b.binary(Kind::Add, res, ins[2], 1, {1});
    } else if (k == "Upsample2x") {
      need(1);
      Shape s = g.shape_of(ins[0]);
      Ref a = b.bcast(ins[0], 3, 2);
      Ref c = b.bcast(a, 5, 2);
      res = b.reshape(c, {s[0], s[1], 2 * s[2], 2 * s[3]});
    } else {
      throw KorchError(KORCH_E_UNSUPPORTED, "no fission rule for operator '" + k + "'");
    }
    out_of[oid] = res.id;
  }
  for (auto& o : j["outputs"].arr) g.outputs.push_back(out_of.at(o.as_int()));
  if (j.has("rewrites") && j["rewrites"].type == Json::Bool && j["rewrites"].b) apply_r1_r3(g);
  return g;
}

Graph parse_primitive_graph(const Json& j) {
  Graph g;
  g.dtype = parse_dtype(j["dtype"].as_str());
  std::map<std::string, int> in_idx;
  for (auto& s : j["inputs"].arr) {
    InputSpec is;
    is.name = s["name"].as_str();
    is.shape = s["shape"].as_ints();
    is.dtype = s.has("dtype") ? parse_dtype(s["dtype"].as_str()) : g.dtype;
    in_idx[is.name] = (int)g.inputs.size();
    g.inputs.push_back(is);
  }
  const auto& nodes = j["nodes"].arr;
  for (size_t i = 0; i < nodes.size(); ++i) {
    const Json& n = nodes[i];
    if (n["id"].as_int() != (int64_t)i) throw KorchError(KORCH_E_PARSE, "primitive ids must be 0..n-1 in order");
    Prim p;
    p.id = (int)i;
    if (!kind_from_name(n["kind"].as_str(), &p.kind))
      throw KorchError(KORCH_E_PARSE, "unknown kind '" + n["kind"].as_str() + "'");
    if (n.has("attrs")) read_prim_attrs(p, n["attrs"]);
    for (auto& r : n["inputs"].arr) {
      if (r.has("node")) p.in.push_back(Ref{false, (int)r["node"].as_int()});
      else p.in.push_back(Ref{true, in_idx.at(r["input"].as_str())});
    }
    p.dtype = g.dtype;
    g.prims.push_back(p);
  }
  for (auto& o : j["outputs"].arr) g.outputs.push_back((int)o.as_int());
  return g;
}
}  // namespace

Graph load_graph(const char* json, size_t n) {
  Json j;
  try {
    j = JsonParser(json, n).parse();
  } catch (JsonError& e) {
    throw KorchError(KORCH_E_PARSE, e.what());
  }
  Graph g;
  try {
    std::string level = j.has("level") ? j["level"].as_str() : "operator";
    if (level == "operator") g = fission_graph(j);
    else if (level == "primitive") g = parse_primitive_graph(j);
    else throw KorchError(KORCH_E_PARSE, "unknown level '" + level + "'");
  } catch (JsonError& e) {
    throw KorchError(KORCH_E_PARSE, e.what());
  }
  g.finalize();
  for (int v : g.topo) {  // (re)infer shapes in topological order
    auto& p = g.prims[v];
    p.shape = infer_shape(g, p);
    for (auto d : p.shape)
      if (d < 1) throw KorchError(KORCH_E_SHAPE, "non-positive extent at primitive " + std::to_string(v));
  }
  if (g.outputs.empty()) throw KorchError(KORCH_E_PARSE, "graph has no outputs");
  for (int o : g.outputs)
    if (o < 0 || o >= (int)g.prims.size()) throw KorchError(KORCH_E_PARSE, "bad output id");
  return g;
}

// ---------------------------------------------------------------- dump / validate
static std::string ints(const std::vector<int64_t>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}
static std::string num(double d) {
  std::ostringstream o;
  o.precision(17);
  o << d;
  return o.str();
}

std::string dump_graph(const Graph& g) {
  std::ostringstream o;
  o << "{\"version\":1,\"level\":\"primitive\",\"dtype\":\"" << dtype_name(g.dtype) << "\",\"inputs\":[";
  for (size_t i = 0; i < g.inputs.size(); ++i)
    o << (i ? "," : "") << "{\"name\":" << json_escape(g.inputs[i].name) << ",\"shape\":" << ints(g.inputs[i].shape)
      << ",\"dtype\":\"" << dtype_name(g.inputs[i].dtype) << "\"}";
  o << "],\"nodes\":[";
  for (size_t i = 0; i < g.prims.size(); ++i) {
    const Prim& p = g.prims[i];
    o << (i ? "," : "") << "{\"id\":" << p.id << ",\"kind\":\"" << kind_name(p.kind) << "\",\"attrs\":{";
    std::vector<std::string> a;
    switch (p.kind) {
      case Kind::AddC: case Kind::MulC: case Kind::DivC: a.push_back("\"c\":" + num(p.c)); break;
      case Kind::Reduce:
        a.push_back("\"axis\":" + std::to_string(p.axis));
        a.push_back(std::string("\"op\":\"") + (p.red == RedOp::Sum ? "sum" : p.red == RedOp::Mean ? "mean" : "max") + "\"");
        break;
      case Kind::Broadcast:
        a.push_back("\"axis\":" + std::to_string(p.axis));
        a.push_back("\"size\":" + std::to_string(p.size));
        break;
      case Kind::Transpose: a.push_back("\"perm\":" + ints(std::vector<int64_t>(p.perm.begin(), p.perm.end()))); break;
      case Kind::Reshape: a.push_back("\"shape\":" + ints(p.new_shape)); break;
      case Kind::Slice:
        a.push_back("\"axis\":" + std::to_string(p.axis));
        a.push_back("\"start\":" + std::to_string(p.start));
        a.push_back("\"end\":" + std::to_string(p.end));
        break;
      case Kind::Pad: {
        std::string s = "\"pads\":[";
        for (size_t k = 0; k < p.pads.size(); ++k)
          s += (k ? "," : "") + std::string("[") + std::to_string(p.pads[k].first) + "," + std::to_string(p.pads[k].second) + "]";
        a.push_back(s + "]");
        a.push_back(std::string("\"mode\":\"") + (p.reflect ? "reflect" : "constant") + "\"");
        a.push_back("\"value\":" + num(p.c));
        break;
      }
      case Kind::Concat: a.push_back("\"axis\":" + std::to_string(p.axis)); break;
      case Kind::Conv2d:
        a.push_back("\"stride\":[" + std::to_string(p.stride[0]) + "," + std::to_string(p.stride[1]) + "]");
        a.push_back("\"pads\":[" + std::to_string(p.cpad[0]) + "," + std::to_string(p.cpad[1]) + "]");
        a.push_back("\"groups\":" + std::to_string(p.groups));
        break;
      case Kind::MaxPool:
        a.push_back("\"k\":" + std::to_string(p.pk));
        a.push_back("\"stride\":" + std::to_string(p.pstride));
        a.push_back("\"pad\":" + std::to_string(p.ppad));
        break;
      case Kind::Constant:
        a.push_back("\"shape\":" + ints(p.new_shape));
        a.push_back("\"value\":" + num(p.c));
        break;
      default: break;
    }
    bool any_port = false;
    std::string pa = "\"port_axes\":{";
    for (size_t s = 0; s < p.port_axes.size(); ++s)
      if (!p.port_axes[s].empty()) {
        pa += (any_port ? "," : "") + std::string("\"") + std::to_string(s) + "\":" +
              ints(std::vector<int64_t>(p.port_axes[s].begin(), p.port_axes[s].end()));
        any_port = true;
      }
    if (any_port) a.push_back(pa + "}");
    for (size_t k = 0; k < a.size(); ++k) o << (k ? "," : "") << a[k];
    o << "},\"inputs\":[";
    for (size_t k = 0; k < p.in.size(); ++k) {
      if (k) o << ",";
      if (p.in[k].is_input) o << "{\"input\":" << json_escape(g.inputs[p.in[k].id].name) << "}";
      else o << "{\"node\":" << p.in[k].id << "}";
    }
    o << "],\"shape\":" << ints(p.shape) << ",\"op\":" << p.op_id << "}";
  }
  o << "],\"outputs\":[";
  for (size_t i = 0; i < g.outputs.size(); ++i) o << (i ? "," : "") << g.outputs[i];
  o << "]}";
  return o.str();
}

std::string validate_graph(const Graph& g) {
  std::string r;
  for (auto& p : g.prims) {
    try {
      if (infer_shape(g, p) != p.shape) r += "primitive " + std::to_string(p.id) + ": inconsistent shape\n";
    } catch (KorchError& e) {
      r += std::string(e.what()) + "\n";
    }
  }
  for (size_t v = 0; v < g.prims.size(); ++v)
    if (g.succs[v].empty() && std::find(g.outputs.begin(), g.outputs.end(), (int)v) == g.outputs.end())
      r += "primitive " + std::to_string(v) + ": dead (no consumer, not an output)\n";
  return r.empty() ? "ok" : r;
}

}  // namespace korch
