// json_lite.hpp — minimal JSON value, parser and writer for the kvsim CLI
// config / report files (reference SPEC.md:444 "JSON with a published
// schema"). Numbers are doubles (integers up to 2^53 are exact); object keys
// keep insertion order so written files are byte-stable.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace jl {

struct Value {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0;
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  static Value number(double d) { Value v; v.kind = Number; v.num = d; return v; }
  static Value string(std::string s) { Value v; v.kind = String; v.str = std::move(s); return v; }
  static Value boolean(bool x) { Value v; v.kind = Bool; v.b = x; return v; }
  static Value array() { Value v; v.kind = Array; return v; }
  static Value object() { Value v; v.kind = Object; return v; }

  bool is_obj() const { return kind == Object; }
  bool is_arr() const { return kind == Array; }
  bool is_num() const { return kind == Number; }
  bool is_str() const { return kind == String; }
  const Value* find(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  Value& set(const std::string& k, Value v) {
    for (auto& kv : obj)
      if (kv.first == k) { kv.second = std::move(v); return kv.second; }
    obj.emplace_back(k, std::move(v));
    return obj.back().second;
  }
  void push(Value v) { arr.push_back(std::move(v)); }
};

struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Value parse() {
    Value v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t i_ = 0;
  [[noreturn]] void fail(const char* what) {
    size_t line = 1;
    for (size_t k = 0; k < i_ && k < s_.size(); ++k) line += s_[k] == '\n';
    throw ParseError(std::string("json: ") + what + " at line " + std::to_string(line));
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r')) ++i_;
  }
  bool lit(const char* w) {
    size_t n = 0;
    while (w[n]) ++n;
    if (s_.compare(i_, n, w) == 0) { i_ += n; return true; }
    return false;
  }
  Value value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    char c = s_[i_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value::string(string());
    if (lit("true")) return Value::boolean(true);
    if (lit("false")) return Value::boolean(false);
    if (lit("null")) return Value();
    if (c == '-' || (c >= '0' && c <= '9')) return number();
    fail("unexpected character");
  }
  Value object() {
    Value v = Value::object();
    ++i_;
    ws();
    if (i_ < s_.size() && s_[i_] == '}') { ++i_; return v; }
    for (;;) {
      ws();
      if (i_ >= s_.size() || s_[i_] != '"') fail("expected key");
      std::string k = string();
      ws();
      if (i_ >= s_.size() || s_[i_] != ':') fail("expected ':'");
      ++i_;
      if (v.find(k)) fail("duplicate key");
      v.obj.emplace_back(k, value());
      ws();
      if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
      if (i_ < s_.size() && s_[i_] == '}') { ++i_; return v; }
      fail("expected ',' or '}'");
    }
  }
  Value array() {
    Value v = Value::array();
    ++i_;
    ws();
    if (i_ < s_.size() && s_[i_] == ']') { ++i_; return v; }
    for (;;) {
      v.arr.push_back(value());
      ws();
      if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
      if (i_ < s_.size() && s_[i_] == ']') { ++i_; return v; }
      fail("expected ',' or ']'");
    }
  }
  std::string string() {
    std::string out;
    ++i_;
    while (i_ < s_.size() && s_[i_] != '"') {
      char c = s_[i_++];
      if (c == '\\') {
        if (i_ >= s_.size()) fail("bad escape");
        char e = s_[i_++];
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (i_ + 4 > s_.size()) fail("bad \\u escape");
            unsigned cp = std::stoul(s_.substr(i_, 4), nullptr, 16);
            i_ += 4;
            if (cp < 0x80) out += (char)cp;
            else if (cp < 0x800) { out += (char)(0xC0 | (cp >> 6)); out += (char)(0x80 | (cp & 63)); }
            else { out += (char)(0xE0 | (cp >> 12)); out += (char)(0x80 | ((cp >> 6) & 63)); out += (char)(0x80 | (cp & 63)); }
            break;
          }
          default: out += e;
        }
      } else {
        out += c;
      }
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  Value number() {
    size_t st = i_;
    if (s_[i_] == '-') ++i_;
    while (i_ < s_.size() && ((s_[i_] >= '0' && s_[i_] <= '9') || s_[i_] == '.' || s_[i_] == 'e' || s_[i_] == 'E' ||
                              s_[i_] == '+' || s_[i_] == '-'))
      ++i_;
    try {
      return Value::number(std::stod(s_.substr(st, i_ - st)));
    } catch (...) {
      fail("bad number");
    }
  }
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

// Shortest round-trip formatting for doubles (%.17g fallback).
inline std::string fmt_num(double d) {
  if (std::isnan(d)) return "null";
  if (std::isinf(d)) return d > 0 ? "1e999" : "-1e999";
  if (d == std::floor(d) && std::fabs(d) < 1e15) {
    char b[32];
    std::snprintf(b, sizeof b, "%.0f", d);
    return b;
  }
  char b[40];
  for (int p = 15; p <= 17; ++p) {
    std::snprintf(b, sizeof b, "%.*g", p, d);
    if (std::stod(b) == d) break;
  }
  return b;
}

inline void escape(std::string& o, const std::string& s) {
  o += '"';
  for (char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\n': o += "\\n"; break;
      case '\t': o += "\\t"; break;
      default:
        if ((unsigned char)c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          o += b;
        } else {
          o += c;
        }
    }
  }
  o += '"';
}

inline void write(std::string& o, const Value& v, int indent = 0, int depth = 0) {
  auto nl = [&](int d) {
    if (indent) {
      o += '\n';
      o.append((size_t)(d * indent), ' ');
    }
  };
  switch (v.kind) {
    case Value::Null: o += "null"; break;
    case Value::Bool: o += v.b ? "true" : "false"; break;
    case Value::Number: o += fmt_num(v.num); break;
    case Value::String: escape(o, v.str); break;
    case Value::Array:
      o += '[';
      for (size_t k = 0; k < v.arr.size(); ++k) {
        if (k) o += ',';
        nl(depth + 1);
        write(o, v.arr[k], indent, depth + 1);
      }
      if (!v.arr.empty()) nl(depth);
      o += ']';
      break;
    case Value::Object:
      o += '{';
      for (size_t k = 0; k < v.obj.size(); ++k) {
        if (k) o += ',';
        nl(depth + 1);
        escape(o, v.obj[k].first);
        o += indent ? ": " : ":";
        write(o, v.obj[k].second, indent, depth + 1);
      }
      if (!v.obj.empty()) nl(depth);
      o += '}';
      break;
  }
}

inline std::string dump(const Value& v, int indent = 2) {
  std::string o;
  write(o, v, indent);
  return o;
}

}  // namespace jl
