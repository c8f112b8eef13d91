// Minimal JSON reader/writer for the graph schema (SPEC S:131-135 + dtype).
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace korch {

struct JsonError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Json {
  enum Type { Null, Bool, Num, Str, Arr, Obj } type = Null;
  bool b = false;
  double num = 0;
  std::string str;
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;

  bool has(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return true;
    return false;
  }
  const Json& operator[](const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return kv.second;
    throw JsonError("missing field '" + k + "'");
  }
  const Json& at(size_t i) const {
    if (type != Arr || i >= arr.size()) throw JsonError("index out of range");
    return arr[i];
  }
  double as_num() const {
    if (type != Num) throw JsonError("expected number");
    return num;
  }
  int64_t as_int() const {
    double v = as_num();
    if (v != (double)(int64_t)v) throw JsonError("expected integer");
    return (int64_t)v;
  }
  const std::string& as_str() const {
    if (type != Str) throw JsonError("expected string");
    return str;
  }
  std::vector<int64_t> as_ints() const {
    if (type != Arr) throw JsonError("expected array");
    std::vector<int64_t> r;
    for (auto& x : arr) r.push_back(x.as_int());
    return r;
  }
};

class JsonParser {
 public:
  JsonParser(const char* s, size_t n) : s_(s), n_(n) {}
  Json parse() {
    Json v = value();
    ws();
    if (p_ != n_) fail("trailing characters");
    return v;
  }

 private:
  const char* s_;
  size_t n_, p_ = 0;
  [[noreturn]] void fail(const std::string& m) {
    throw JsonError("JSON parse error at byte " + std::to_string(p_) + ": " + m);
  }
  void ws() {
    while (p_ < n_ && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\t' || s_[p_] == '\r')) ++p_;
  }
  char peek() {
    ws();
    if (p_ >= n_) fail("unexpected end");
    return s_[p_];
  }
  void expect(char c) {
    if (peek() != c) fail(std::string("expected '") + c + "'");
    ++p_;
  }
  Json value() {
    char c = peek();
    Json v;
    if (c == '{') {
      v.type = Json::Obj;
      ++p_;
      if (peek() == '}') { ++p_; return v; }
      for (;;) {
        Json k = string_();
        expect(':');
        v.obj.emplace_back(k.str, value());
        char d = peek();
        ++p_;
        if (d == '}') break;
        if (d != ',') fail("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.type = Json::Arr;
      ++p_;
      if (peek() == ']') { ++p_; return v; }
      for (;;) {
        v.arr.push_back(value());
        char d = peek();
        ++p_;
        if (d == ']') break;
        if (d != ',') fail("expected ',' or ']'");
      }
    } else if (c == '"') {
      v = string_();
    } else if (c == 't' || c == 'f' || c == 'n') {
      auto lit = [&](const char* w) {
        size_t l = strlen_(w);
        if (p_ + l > n_ || std::string(s_ + p_, l) != w) fail("bad literal");
        p_ += l;
      };
      if (c == 't') { lit("true"); v.type = Json::Bool; v.b = true; }
      else if (c == 'f') { lit("false"); v.type = Json::Bool; v.b = false; }
      else { lit("null"); v.type = Json::Null; }
    } else {
      size_t st = p_;
      while (p_ < n_ && (isdigit_(s_[p_]) || s_[p_] == '-' || s_[p_] == '+' || s_[p_] == '.' ||
                         s_[p_] == 'e' || s_[p_] == 'E'))
        ++p_;
      if (st == p_) fail("unexpected character");
      v.type = Json::Num;
      v.num = std::stod(std::string(s_ + st, p_ - st));
    }
    return v;
  }
  static size_t strlen_(const char* w) { size_t l = 0; while (w[l]) ++l; return l; }
  static bool isdigit_(char c) { return c >= '0' && c <= '9'; }
  Json string_() {
    expect('"');
    Json v;
    v.type = Json::Str;
    while (p_ < n_ && s_[p_] != '"') {
      if (s_[p_] == '\\') {
        ++p_;
        if (p_ >= n_) fail("bad escape");
        char e = s_[p_];
        if (e == 'n') v.str += '\n';
        else if (e == 't') v.str += '\t';
        else if (e == 'u') { p_ += 4; v.str += '?'; }
        else v.str += e;
        ++p_;
      } else {
        v.str += s_[p_++];
      }
    }
    if (p_ >= n_) fail("unterminated string");
    ++p_;
    return v;
  }
};

inline std::string json_escape(const std::string& s) {
  std::string r = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') { r += '\\'; r += c; }
    else if (c == '\n') r += "\\n";
    else r += c;
  }
  return r + "\"";
}

}  // namespace korch
