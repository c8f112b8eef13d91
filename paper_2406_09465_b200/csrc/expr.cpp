#include "expr.h"

#include <stdexcept>

namespace korch {

static int64_t floordiv(int64_t a, int64_t b) { int64_t q = a / b; if ((a % b) && ((a < 0) != (b < 0))) --q; return q; }
static int64_t floormod(int64_t a, int64_t b) { int64_t m = a % b; if (m && ((m < 0) != (b < 0))) m += b; return m; }

int64_t Lin::lo() const {
  int64_t r = c0;
  for (auto& t : terms) r += t.first > 0 ? t.first * t.second.lo : t.first * t.second.hi;
  return r;
}
int64_t Lin::hi() const {
  int64_t r = c0;
  for (auto& t : terms) r += t.first > 0 ? t.first * t.second.hi : t.first * t.second.lo;
  return r;
}
std::string Lin::key() const {
  std::string s = std::to_string(c0);
  for (auto& t : terms) s += "+" + std::to_string(t.first) + "*" + t.second.key;
  return s;
}

Lin ExprCtx::from_atom(Atom at, int64_t coef) const {
  Lin l;
  if (coef) l.terms.push_back({coef, std::move(at)});
  return l;
}

Lin ExprCtx::var(int v) const {
  Atom a;
  a.type = Atom::Var;
  a.var = v;
  a.lo = vars[v].lo;
  a.hi = vars[v].hi;
  a.key = "v" + std::to_string(v);
  if (a.lo == a.hi) return cst(a.lo);
  return from_atom(a);
}

Lin ExprCtx::code(const std::string& c, int64_t lo, int64_t hi) const {
  Atom a;
  a.type = Atom::Code;
  a.code = c;
  a.lo = lo;
  a.hi = hi;
  a.key = "{" + c + "}";
  return from_atom(a);
}

// c*k*(X / c) + k*(X % c) == k*X (non-negative X): folds the index arithmetic that a
// reshape followed by its inverse leaves behind (e.g. a row axis merged from two axes).
static Lin recombine(const Lin& r) {
  for (size_t i = 0; i < r.terms.size(); ++i) {
    const Atom& d = r.terms[i].second;
    if (d.type != Atom::Div || r.terms[i].first % d.c) continue;
    const int64_t k = r.terms[i].first / d.c;
    const std::string sk = d.sub->key();
    for (size_t j = 0; j < r.terms.size(); ++j) {
      const Atom& m = r.terms[j].second;
      if (j == i || m.type != Atom::Mod || m.c != d.c || r.terms[j].first != k || m.sub->key() != sk) continue;
      if (d.sub->lo() < 0) continue;
      Lin rest;
      rest.c0 = r.c0;
      for (size_t t = 0; t < r.terms.size(); ++t)
        if (t != i && t != j) rest.terms.push_back(r.terms[t]);
      return ExprCtx::add(rest, ExprCtx::scale(*d.sub, k));
    }
  }
  return r;
}

Lin ExprCtx::add(const Lin& a, const Lin& b) {
  Lin r;
  r.c0 = a.c0 + b.c0;
  size_t i = 0, j = 0;
  while (i < a.terms.size() || j < b.terms.size()) {
    if (j >= b.terms.size() || (i < a.terms.size() && a.terms[i].second.key < b.terms[j].second.key)) {
      r.terms.push_back(a.terms[i++]);
    } else if (i >= a.terms.size() || b.terms[j].second.key < a.terms[i].second.key) {
      r.terms.push_back(b.terms[j++]);
    } else {
      int64_t c = a.terms[i].first + b.terms[j].first;
      if (c) r.terms.push_back({c, a.terms[i].second});
      ++i, ++j;
    }
  }
  return recombine(r);
}

Lin ExprCtx::scale(const Lin& a, int64_t k) {
  Lin r;
  if (!k) return r;
  r.c0 = a.c0 * k;
  for (auto& t : a.terms) r.terms.push_back({t.first * k, t.second});
  return r;
}

// Split a = c*Q + R where Q gathers the terms whose coefficient is a multiple of c.
static void split(const Lin& a, int64_t c, Lin* Q, Lin* R) {
  *Q = Lin();
  *R = Lin();
  for (auto& t : a.terms) {
    if (t.first % c == 0) Q->terms.push_back({t.first / c, t.second});
    else R->terms.push_back(t);
  }
  int64_t rc = floormod(a.c0, c);
  Q->c0 = floordiv(a.c0 - rc, c);
  R->c0 = rc;
}

Lin ExprCtx::div(const Lin& a, int64_t c) const {
  if (c == 1) return a;
  if (a.is_const()) return cst(floordiv(a.c0, c));
  Lin Q, R;
  split(a, c, &Q, &R);
  int64_t rl = R.lo(), rh = R.hi();
  if (rl >= 0 && rh < c) return Q;                    // R contributes nothing
  if (rl >= 0) {                                       // Q + floor(R / c)
    if (floordiv(rl, c) == floordiv(rh, c)) return add(Q, cst(floordiv(rl, c)));
    Atom at;
    at.type = Atom::Div;
    at.sub = std::make_shared<Lin>(R);
    at.c = c;
    at.lo = floordiv(rl, c);
    at.hi = floordiv(rh, c);
    at.key = "(" + R.key() + ")/" + std::to_string(c);
    return add(Q, from_atom(at));
  }
  Atom at;  // negative parts: keep whole (only reached in masked pad regions)
  at.type = Atom::Div;
  at.sub = std::make_shared<Lin>(a);
  at.c = c;
  at.lo = floordiv(a.lo(), c);
  at.hi = floordiv(a.hi(), c);
  at.key = "(" + a.key() + ")/" + std::to_string(c);
  return from_atom(at);
}

Lin ExprCtx::mod(const Lin& a, int64_t c) const {
  if (c == 1) return cst(0);
  if (a.is_const()) return cst(floormod(a.c0, c));
  Lin Q, R;
  split(a, c, &Q, &R);
  int64_t rl = R.lo(), rh = R.hi();
  if (rl >= 0 && rh < c) return R;
  const Lin& base = rl >= 0 ? R : a;
  Atom at;
  at.type = Atom::Mod;
  at.sub = std::make_shared<Lin>(base);
  at.c = c;
  at.lo = 0;
  at.hi = c - 1;
  at.key = "(" + base.key() + ")%" + std::to_string(c);
  return from_atom(at);
}

std::string ExprCtx::emit(const Lin& a, const std::map<int, std::string>* ov) const {
  std::string s;
  for (auto& t : a.terms) {
    std::string at;
    const Atom& x = t.second;
    switch (x.type) {
      case Atom::Var: {
        if (ov && ov->count(x.var)) at = "(" + ov->at(x.var) + ")";
        else at = vars[x.var].name;
        break;
      }
      case Atom::Div: at = "((" + emit(*x.sub, ov) + ")/" + std::to_string(x.c) + ")"; break;
      case Atom::Mod: at = "((" + emit(*x.sub, ov) + ")%" + std::to_string(x.c) + ")"; break;
      case Atom::Code: at = "(" + x.code + ")"; break;
    }
    if (!s.empty()) s += " + ";
    s += t.first == 1 ? at : std::to_string(t.first) + "*" + at;
  }
  if (a.c0 || s.empty()) {
    if (!s.empty()) s += " + ";
    s += std::to_string(a.c0);
  }
  return s;
}

static bool atom_mentions(const Atom& a, int v) {
  if (a.type == Atom::Var) return a.var == v;
  if (a.type == Atom::Code) return a.code.find("/*v" + std::to_string(v) + "*/") != std::string::npos;
  for (auto& t : a.sub->terms)
    if (atom_mentions(t.second, v)) return true;
  return false;
}

bool ExprCtx::linear_in(const Lin& a, int v, int64_t* coef) {
  *coef = 0;
  for (auto& t : a.terms) {
    if (t.second.type == Atom::Var && t.second.var == v) *coef = t.first;
    else if (atom_mentions(t.second, v)) return false;
  }
  return true;
}

bool ExprCtx::depends_on(const Lin& a, int v) {
  for (auto& t : a.terms)
    if (atom_mentions(t.second, v)) return true;
  return false;
}

bool ExprCtx::rest_divisible(const Lin& a, int v, int64_t k) {
  if (a.c0 % k) return false;
  for (auto& t : a.terms) {
    if (t.second.type == Atom::Var && t.second.var == v) continue;
    if (t.first % k) return false;
  }
  return true;
}

Lin ExprCtx::subst(const Lin& a, int v, const Lin& e) const {
  Lin r = cst(a.c0);
  for (auto& t : a.terms) {
    const Atom& x = t.second;
    Lin piece;
    if (x.type == Atom::Var && x.var == v) piece = e;
    else if ((x.type == Atom::Div || x.type == Atom::Mod) && atom_mentions(x, v)) {
      Lin s = subst(*x.sub, v, e);
      piece = x.type == Atom::Div ? div(s, x.c) : mod(s, x.c);
    } else {
      piece = from_atom(x);
    }
    r = add(r, scale(piece, t.first));
  }
  return r;
}

}  // namespace korch
