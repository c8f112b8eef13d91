// Primitive-graph rewrites R1-R3 (Fig. 2b), the TASO transformations the
// paper applies at a Softmax feeding a MatMul:
//   R1  ReduceSum(e, last) -> Reshape(MatMul(e, C_s)), C_s a constant of ones  (P:225, P:227 fn.)
//   R2  MatMul(Div(e, Bcast(x)), V) -> Div(MatMul(e, V), Bcast(x))
//   R3  MatMul(e, V) and MatMul(e, C_s) -> MatMul(e, Pad(V, 16 ones columns)),
//       then Slice(num) and Slice(den)                                       (reading A28)
// Afterwards primitives are renumbered by Kahn's algorithm, smallest pre-renumbering id
// first (new primitives get ids after all existing ones, in creation order).
#include <algorithm>
#include <array>
#include <map>
#include <queue>
#include <set>

#include "../../include/korch.h"
#include "ir.h"

namespace korch {

namespace {
struct Work {
  Graph& g;
  std::map<int, Prim> P;
  std::vector<int> outputs;
  int next = 0;
  explicit Work(Graph& gg) : g(gg) {
    for (auto& p : g.prims) P[p.id] = p;
    outputs = g.outputs;
    next = (int)g.prims.size();
  }
  const Shape& shape(const Ref& r) const { return r.is_input ? g.inputs[r.id].shape : P.at(r.id).shape; }
  std::vector<int> consumers(int id) const {
    std::vector<int> c;
    for (auto& kv : P)
      for (auto& r : kv.second.in)
        if (!r.is_input && r.id == id) {
          c.push_back(kv.first);
          break;
        }
    return c;
  }
  Ref add(Prim p, std::vector<Ref> in, int op) {
    p.id = next++;
    p.in = std::move(in);
    p.dtype = g.dtype;
    p.op_id = op;
    // shape inference needs a Graph view: temporarily resolve inputs here
    p.shape = infer(p);
    P[p.id] = p;
    return Ref{false, p.id};
  }
  Shape infer(const Prim& p) {
    switch (p.kind) {
      case Kind::Constant: return p.new_shape;
      case Kind::MatMul: {
        const Shape &a = shape(p.in[0]), &b = shape(p.in[1]);
        Shape r(a.begin(), a.end() - 1);
        r.push_back(b.back());
        return r;
      }
      case Kind::Reshape: return p.new_shape;
      case Kind::Broadcast: {
        Shape s = shape(p.in[0]);
        s.insert(s.begin() + p.axis, p.size);
        return s;
      }
      case Kind::Div: return shape(p.in[0]);
      case Kind::Pad: {
        Shape s = shape(p.in[0]);
        for (size_t i = 0; i < s.size(); ++i) s[i] += p.pads[i].first + p.pads[i].second;
        return s;
      }
      case Kind::Slice: {
        Shape s = shape(p.in[0]);
        s[p.axis] = p.end - p.start;
        return s;
      }
      default: throw KorchError(KORCH_E_UNSUPPORTED, "rewrite produced an unexpected primitive");
    }
  }
  void replace_uses(int old, Ref nw) {
    for (auto& kv : P)
      for (auto& r : kv.second.in)
        if (!r.is_input && r.id == old) r = nw;
    for (auto& o : outputs)
      if (o == old) o = nw.id;
  }
  void remove_dead() {
    bool changed = true;
    while (changed) {
      changed = false;
      for (auto it = P.begin(); it != P.end();) {
        int v = it->first;
        if (std::find(outputs.begin(), outputs.end(), v) == outputs.end() && consumers(v).empty()) {
          it = P.erase(it);
          changed = true;
        } else {
          ++it;
        }
      }
    }
  }
};

bool same_ref(const Ref& a, const Ref& b) { return a.is_input == b.is_input && a.id == b.id; }
}  // namespace

void apply_r1_r3(Graph& g) {
  Work w(g);
  // sites: r = reduce_sum(e, last), b = bcast(r, last), p = div(e, b), o = matmul(p, V)
  std::vector<std::array<int, 4>> sites;
  for (auto& kv : w.P) {
    const Prim& r = kv.second;
    if (r.kind != Kind::Reduce || r.red != RedOp::Sum || r.in[0].is_input) continue;
    const Shape& se = w.shape(r.in[0]);
    if (se.size() < 2 || r.axis != (int)se.size() - 1) continue;
    auto cb = w.consumers(r.id);
    if (cb.size() != 1 || w.P[cb[0]].kind != Kind::Broadcast || w.P[cb[0]].axis != (int)se.size() - 1) continue;
    auto cp = w.consumers(cb[0]);
    if (cp.size() != 1 || w.P[cp[0]].kind != Kind::Div) continue;
    const Prim& p = w.P[cp[0]];
    if (!same_ref(p.in[0], r.in[0]) || p.in[1].is_input || p.in[1].id != cb[0]) continue;
    auto co = w.consumers(p.id);
    if (co.size() != 1 || w.P[co[0]].kind != Kind::MatMul) continue;
    if (std::find(w.outputs.begin(), w.outputs.end(), p.id) != w.outputs.end()) continue;
    const Prim& o = w.P[co[0]];
    if (o.in[0].is_input || o.in[0].id != p.id) continue;
    sites.push_back({r.id, cb[0], p.id, o.id});
  }
  for (auto& s : sites) {
    Prim r = w.P.at(s[0]), p = w.P.at(s[2]), o = w.P.at(s[3]);
    Ref e = r.in[0];
    Shape se = w.shape(e);
    int64_t n = se.back();
    int last = (int)se.size() - 1;
    // R1
    Prim cs; cs.kind = Kind::Constant; cs.new_shape = {n, 1}; cs.c = 1.0;
    Ref cref = w.add(cs, {}, r.op_id);
    Prim m2p; m2p.kind = Kind::MatMul;
    Ref m2 = w.add(m2p, {e, cref}, r.op_id);
    Prim r1p; r1p.kind = Kind::Reshape; r1p.new_shape = Shape(se.begin(), se.end() - 1);
    Ref r1 = w.add(r1p, {m2}, r.op_id);
    w.replace_uses(r.id, r1);
    // R2
    Ref v = o.in[1];
    int64_t nv = w.shape(v).back();
    Prim m1p; m1p.kind = Kind::MatMul;
    Ref m1 = w.add(m1p, {e, v}, o.op_id);
    Prim bxp; bxp.kind = Kind::Broadcast; bxp.axis = last; bxp.size = nv;
    Ref bx = w.add(bxp, {r1}, p.op_id);
    Prim dp; dp.kind = Kind::Div;
    Ref d = w.add(dp, {m1, bx}, p.op_id);
    w.replace_uses(o.id, d);
    // R3
    const Shape& sv = w.shape(v);
    Prim vhp; vhp.kind = Kind::Pad; vhp.c = 1.0;
    for (size_t i = 0; i < sv.size(); ++i) vhp.pads.push_back({0, i + 1 == sv.size() ? 16 : 0});
    Ref vh = w.add(vhp, {v}, o.op_id);
    Prim mmp; mmp.kind = Kind::MatMul;
    Ref mm = w.add(mmp, {e, vh}, o.op_id);
    Prim nump; nump.kind = Kind::Slice; nump.axis = last; nump.start = 0; nump.end = nv;
    Ref num = w.add(nump, {mm}, o.op_id);
    Prim denp; denp.kind = Kind::Slice; denp.axis = last; denp.start = nv; denp.end = nv + 1;
    Ref den = w.add(denp, {mm}, r.op_id);
    w.replace_uses(m1.id, num);
    w.replace_uses(m2.id, den);
    w.remove_dead();
  }
  // renumber: Kahn, smallest old id first
  std::map<int, int> indeg;
  std::map<int, std::vector<int>> users;
  for (auto& kv : w.P) {
    std::set<int> deps;
    for (auto& r : kv.second.in)
      if (!r.is_input) deps.insert(r.id);
    indeg[kv.first] = (int)deps.size();
    for (int d : deps) users[d].push_back(kv.first);
  }
  std::priority_queue<int, std::vector<int>, std::greater<int>> pq;
  for (auto& kv : indeg)
    if (!kv.second) pq.push(kv.first);
  std::map<int, int> nid;
  std::vector<int> order;
  while (!pq.empty()) {
    int v = pq.top();
    pq.pop();
    nid[v] = (int)order.size();
    order.push_back(v);
    for (int u : users[v])
      if (--indeg[u] == 0) pq.push(u);
  }
  std::vector<Prim> prims;
  for (int old : order) {
    Prim p = w.P[old];
    p.id = nid[old];
    for (auto& r : p.in)
      if (!r.is_input) r.id = nid[r.id];
    prims.push_back(p);
  }
  g.prims = prims;
  g.outputs.clear();
  for (int o : w.outputs) g.outputs.push_back(nid[o]);
}

}  // namespace korch
