// Minimal JSON value/parser/writer used at the C-ABI boundary: graph
// descriptions, partition rules, strategy specs and plan dumps cross the
// boundary as UTF-8 JSON documents ("Graph description format is
// a declarative JSON document"). Integers are kept exact (int64/uint64).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace opflow::json {

struct Value;
using Array = std::vector<Value>;
using Object = std::vector<std::pair<std::string, Value>>;

struct Value {
  enum class T { Null, Bool, Int, Double, String, Array, Object } t = T::Null;
  bool b = false;
  int64_t i = 0;
  uint64_t u = 0;      // exact unsigned view of an integer literal
  bool is_neg = false;
  double d = 0.0;
  std::string s;
  std::shared_ptr<Array> a;
  std::shared_ptr<Object> o;

  bool is_null() const { return t == T::Null; }
  bool is_num() const { return t == T::Int || t == T::Double; }
  double num() const { return t == T::Int ? static_cast<double>(i) : d; }
  int64_t as_i64() const {
    if (t == T::Int) return i;
    if (t == T::Double) return static_cast<int64_t>(d);
    throw std::runtime_error("json: expected integer");
  }
  uint64_t as_u64() const {
    if (t == T::Int) return is_neg ? static_cast<uint64_t>(i) : u;
    throw std::runtime_error("json: expected unsigned integer");
  }
  const std::string& str() const {
    if (t != T::String) throw std::runtime_error("json: expected string");
    return s;
  }
  const Array& arr() const {
    if (t != T::Array) throw std::runtime_error("json: expected array");
    return *a;
  }
  const Object& obj() const {
    if (t != T::Object) throw std::runtime_error("json: expected object");
    return *o;
  }
  const Value* get(const std::string& key) const {
    if (t != T::Object) return nullptr;
    for (const auto& kv : *o)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& text) : s_(text) {}
  Value parse() {
    Value v = value();
    ws();
    if (p_ != s_.size()) err("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  std::size_t p_ = 0;

  [[noreturn]] void err(const char* what) {
    throw std::runtime_error(std::string("json parse error at ") + std::to_string(p_) + ": " +
                             what);
  }
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\t' || s_[p_] == '\r'))
      ++p_;
  }
  bool lit(const char* w) {
    std::size_t n = 0;
    while (w[n]) ++n;
    if (s_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (p_ >= s_.size()) err("unexpected end");
    char c = s_[p_];
    Value v;
    if (c == '{') {
      ++p_;
      v.t = Value::T::Object;
      v.o = std::make_shared<Object>();
      ws();
      if (p_ < s_.size() && s_[p_] == '}') {
        ++p_;
        return v;
      }
      for (;;) {
        ws();
        if (p_ >= s_.size() || s_[p_] != '"') err("expected key");
        std::string k = string();
        ws();
        if (p_ >= s_.size() || s_[p_] != ':') err("expected ':'");
        ++p_;
        v.o->emplace_back(std::move(k), value());
        ws();
        if (p_ < s_.size() && s_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < s_.size() && s_[p_] == '}') {
          ++p_;
          return v;
        }
        err("expected ',' or '}'");
      }
    }
    if (c == '[') {
      ++p_;
      v.t = Value::T::Array;
      v.a = std::make_shared<Array>();
      ws();
      if (p_ < s_.size() && s_[p_] == ']') {
        ++p_;
        return v;
      }
      for (;;) {
        v.a->push_back(value());
        ws();
        if (p_ < s_.size() && s_[p_] == ',') {
          ++p_;
          continue;
        }
        if (p_ < s_.size() && s_[p_] == ']') {
          ++p_;
          return v;
        }
        err("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.t = Value::T::String;
      v.s = string();
      return v;
    }
    if (lit("true")) {
      v.t = Value::T::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.t = Value::T::Bool;
      return v;
    }
    if (lit("null")) return v;
    return number();
  }
  std::string string() {
    ++p_;  // opening quote
    std::string out;
    while (p_ < s_.size() && s_[p_] != '"') {
      char c = s_[p_++];
      if (c == '\\') {
        if (p_ >= s_.size()) err("bad escape");
        char e = s_[p_++];
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (p_ + 4 > s_.size()) err("bad \\u escape");
            unsigned cp = std::stoul(s_.substr(p_, 4), nullptr, 16);
            p_ += 4;
            if (cp < 0x80) {
              out += static_cast<char>(cp);
            } else if (cp < 0x800) {
              out += static_cast<char>(0xC0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              out += static_cast<char>(0xE0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: out += e; break;
        }
      } else {
        out += c;
      }
    }
    if (p_ >= s_.size()) err("unterminated string");
    ++p_;
    return out;
  }
  Value number() {
    std::size_t start = p_;
    bool neg = false, is_int = true;
    if (s_[p_] == '-') {
      neg = true;
      ++p_;
    }
    while (p_ < s_.size()) {
      char c = s_[p_];
      if (c >= '0' && c <= '9') {
        ++p_;
      } else if (c == '.' || c == 'e' || c == 'E' || c == '+' || (c == '-' && p_ > start)) {
        is_int = false;
        ++p_;
      } else {
        break;
      }
    }
    if (p_ == start || (neg && p_ == start + 1)) err("bad number");
    std::string tok = s_.substr(start, p_ - start);
    Value v;
    if (is_int) {
      v.t = Value::T::Int;
      v.is_neg = neg;
      if (neg) {
        v.i = std::stoll(tok);
        v.u = static_cast<uint64_t>(v.i);
      } else {
        v.u = std::stoull(tok);
        v.i = static_cast<int64_t>(v.u);
      }
      v.d = neg ? static_cast<double>(v.i) : static_cast<double>(v.u);
    } else {
      v.t = Value::T::Double;
      v.d = std::strtod(tok.c_str(), nullptr);
    }
    return v;
  }
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

inline std::string quote(const std::string& s) {
  std::string out = "\"";
  for (char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\t': out += "\\t"; break;
      default: out += c;
    }
  }
  out += '"';
  return out;
}

template <class T>
std::string int_list(const std::vector<T>& v) {
  std::string out = "[";
  for (std::size_t i = 0; i < v.size(); ++i) {
    if (i) out += ',';
    out += std::to_string(v[i]);
  }
  out += ']';
  return out;
}

inline std::string str_list(const std::vector<std::string>& v) {
  std::string out = "[";
  for (std::size_t i = 0; i < v.size(); ++i) {
    if (i) out += ',';
    out += quote(v[i]);
  }
  out += ']';
  return out;
}

}  // namespace opflow::json
