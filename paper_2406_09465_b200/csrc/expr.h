// Quasi-affine index expressions: const + sum(coef * atom), atoms = variables,
// floor-div / mod of a sub-expression by a positive constant, or opaque code.
// Layout primitives (O[x] = I[L(x)]) compose as substitutions on these;
// the simplifier removes the div/mod pairs that reshape split/merge chains create,
// so the generated address arithmetic stays linear where it can, and the vectoriser
// can ask "is this address j + (multiple of V)?".
#pragma once
#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace korch {

struct Lin;
struct Atom {
  enum Type { Var, Div, Mod, Code } type = Var;
  int var = -1;                 // Var
  std::shared_ptr<Lin> sub;     // Div / Mod operand
  int64_t c = 1;                // Div / Mod constant
  std::string code;             // Code (opaque C expression)
  int64_t lo = 0, hi = 0;       // value range (inclusive)
  std::string key;              // canonical text
};

struct Lin {
  int64_t c0 = 0;
  std::vector<std::pair<int64_t, Atom>> terms;  // sorted by atom key, coef != 0
  int64_t lo() const;
  int64_t hi() const;
  std::string key() const;
  bool is_const() const { return terms.empty(); }
};

struct VarInfo {
  std::string name;
  int64_t lo, hi;
};

class ExprCtx {
 public:
  std::vector<VarInfo> vars;
  int add_var(const std::string& name, int64_t lo, int64_t hi) {
    vars.push_back({name, lo, hi});
    return (int)vars.size() - 1;
  }
  Lin var(int v) const;
  static Lin cst(int64_t c) { Lin l; l.c0 = c; return l; }
  Lin code(const std::string& code, int64_t lo, int64_t hi) const;
  static Lin add(const Lin& a, const Lin& b);
  static Lin scale(const Lin& a, int64_t k);
  Lin div(const Lin& a, int64_t c) const;
  Lin mod(const Lin& a, int64_t c) const;
  // C code; var names come from `vars` unless overridden (var id -> text)
  std::string emit(const Lin& a, const std::map<int, std::string>* ov = nullptr) const;
  // coefficient of variable v if v only appears linearly; returns false if v
  // appears inside a div/mod/code atom.
  static bool linear_in(const Lin& a, int v, int64_t* coef);
  static bool depends_on(const Lin& a, int v);
  // all coefficients except var v's, and the constant, divisible by k?
  static bool rest_divisible(const Lin& a, int v, int64_t k);
  // substitute variable v by expression e
  Lin subst(const Lin& a, int v, const Lin& e) const;

 private:
  Lin from_atom(Atom at, int64_t coef = 1) const;
};

}  // namespace korch
