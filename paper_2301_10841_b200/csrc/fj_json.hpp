// Minimal JSON value + parser/emitter for the plan-file dialect of
// SPEC.md:171 ("query-ir External Interfaces") and SPEC.md:255.
// Only what the dialect needs: null, bool, integer/float numbers, strings
// (with \" \\ \n \t \uXXXX-as-ASCII escapes), arrays and objects.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "fj_errors.hpp"

namespace fj {
namespace json {

struct Value {
  enum class Kind { Null, Bool, Number, String, Array, Object };
  Kind kind = Kind::Null;
  bool b = false;
  double num = 0;
  std::string str;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;  // insertion order kept

  bool is_string() const { return kind == Kind::String; }
  bool is_array() const { return kind == Kind::Array; }
  bool is_object() const { return kind == Kind::Object; }
  const Value* find(const std::string& k) const {
    for (auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  const Value& at(const std::string& k) const {
    const Value* v = find(k);
    if (!v) throw ParseError("missing key '" + k + "'");
    return *v;
  }
  static Value string(std::string s) {
    Value v;
    v.kind = Kind::String;
    v.str = std::move(s);
    return v;
  }
  static Value array() {
    Value v;
    v.kind = Kind::Array;
    return v;
  }
  static Value object() {
    Value v;
    v.kind = Kind::Object;
    return v;
  }
  static Value number(double d) {
    Value v;
    v.kind = Kind::Number;
    v.num = d;
    return v;
  }
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

  [[noreturn]] void fail(const std::string& why) {
    throw ParseError("json: " + why + " at offset " + std::to_string(i_));
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\t' || s_[i_] == '\r')) ++i_;
  }
  char peek() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    return s_[i_];
  }
  void expect(char c) {
    if (peek() != c) fail(std::string("expected '") + c + "'");
    ++i_;
  }
  Value value() {
    char c = peek();
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value::string(string());
    if (s_.compare(i_, 4, "null") == 0) {
      i_ += 4;
      return Value();
    }
    if (s_.compare(i_, 4, "true") == 0) {
      i_ += 4;
      Value v;
      v.kind = Value::Kind::Bool;
      v.b = true;
      return v;
    }
    if (s_.compare(i_, 5, "false") == 0) {
      i_ += 5;
      Value v;
      v.kind = Value::Kind::Bool;
      return v;
    }
    if (c == '-' || (c >= '0' && c <= '9')) return number();
    fail("unexpected character");
  }
  Value number() {
    size_t st = i_;
    if (s_[i_] == '-') ++i_;
    while (i_ < s_.size() && (isdigit((unsigned char)s_[i_]) || s_[i_] == '.' || s_[i_] == 'e' ||
                              s_[i_] == 'E' || s_[i_] == '+' || s_[i_] == '-'))
      ++i_;
    return Value::number(std::stod(s_.substr(st, i_ - st)));
  }
  std::string string() {
    expect('"');
    std::string out;
    while (true) {
      if (i_ >= s_.size()) fail("unterminated string");
      char c = s_[i_++];
      if (c == '"') break;
      if (c == '\\') {
        if (i_ >= s_.size()) fail("bad escape");
        char e = s_[i_++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (i_ + 4 > s_.size()) fail("bad \\u escape");
            unsigned cp = std::stoul(s_.substr(i_, 4), nullptr, 16);
            i_ += 4;
            if (cp > 0x7f) fail("non-ASCII \\u escape unsupported");
            out += char(cp);
            break;
          }
          default: fail("bad escape");
        }
      } else {
        out += c;
      }
    }
    return out;
  }
  Value array() {
    expect('[');
    Value v = Value::array();
    if (peek() == ']') {
      ++i_;
      return v;
    }
    while (true) {
      v.arr.push_back(value());
      char c = peek();
      ++i_;
      if (c == ']') break;
      if (c != ',') fail("expected ',' or ']'");
    }
    return v;
  }
  Value object() {
    expect('{');
    Value v = Value::object();
    if (peek() == '}') {
      ++i_;
      return v;
    }
    while (true) {
      if (peek() != '"') fail("expected key");
      std::string k = string();
      expect(':');
      v.obj.emplace_back(k, value());
      char c = peek();
      ++i_;
      if (c == '}') break;
      if (c != ',') fail("expected ',' or '}'");
    }
    return v;
  }
};

inline Value parse(const std::string& s) { return Parser(s).parse(); }

inline std::string quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') {
      o += '\\';
      o += c;
    } else if (c == '\n') {
      o += "\\n";
    } else {
      o += c;
    }
  }
  return o + "\"";
}

inline std::string dump(const Value& v) {
  switch (v.kind) {
    case Value::Kind::Null: return "null";
    case Value::Kind::Bool: return v.b ? "true" : "false";
    case Value::Kind::Number: {
      if (v.num == (double)(int64_t)v.num) return std::to_string((int64_t)v.num);
      return std::to_string(v.num);
    }
    case Value::Kind::String: return quote(v.str);
    case Value::Kind::Array: {
      std::string o = "[";
      for (size_t i = 0; i < v.arr.size(); ++i) {
        if (i) o += ",";
        o += dump(v.arr[i]);
      }
      return o + "]";
    }
    case Value::Kind::Object: {
      std::string o = "{";
      for (size_t i = 0; i < v.obj.size(); ++i) {
        if (i) o += ",";
        o += quote(v.obj[i].first) + ":" + dump(v.obj[i].second);
      }
      return o + "}";
    }
  }
  return "null";
}

}  // namespace json
}  // namespace fj
