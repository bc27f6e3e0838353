// Minimal JSON reader for chain files (the writer is json_writer.hpp): null, booleans,
// numbers (integers kept exact), strings with the standard escapes, arrays and objects.
// Object members iterate in key order, as the reference's nlohmann::json objects do
// (proj/src/chain_file.cpp iterates "writes" that way).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "ooc/core.hpp"

namespace ooc {

struct JsonValue {
  enum Kind { null, boolean, number, string, array, object } kind = null;
  bool b = false;
  double num = 0.0;
  bool is_int = false;
  long long inum = 0;
  std::string str;
  std::vector<JsonValue> arr;
  std::map<std::string, JsonValue> obj;

  bool has(const std::string& k) const { return kind == object && obj.count(k) > 0; }
  const JsonValue& at(const std::string& k) const {
    auto it = kind == object ? obj.find(k) : obj.end();
    if (it == obj.end()) throw ValidationError("chain file: missing key '" + k + "'");
    return it->second;
  }
  long long as_int() const {
    if (kind != number) throw ValidationError("chain file: expected a number");
    return is_int ? inum : static_cast<long long>(num);
  }
  double as_double() const {
    if (kind != number) throw ValidationError("chain file: expected a number");
    return num;
  }
  const std::string& as_string() const {
    if (kind != string) throw ValidationError("chain file: expected a string");
    return str;
  }
};

class JsonParser {
 public:
  explicit JsonParser(const std::string& t) : t_(t) {}
  JsonValue parse() {
    JsonValue v = value();
    ws();
    if (i_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& m) const {
    throw ValidationError("chain file: JSON parse error at offset " + std::to_string(i_) + ": " + m);
  }
  void ws() {
    while (i_ < t_.size() && (t_[i_] == ' ' || t_[i_] == '\t' || t_[i_] == '\n' || t_[i_] == '\r')) ++i_;
  }
  bool eat(char c) {
    ws();
    if (i_ < t_.size() && t_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  bool word(const char* w) {
    const std::size_t n = std::char_traits<char>::length(w);
    if (t_.compare(i_, n, w) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  JsonValue value() {
    ws();
    if (i_ >= t_.size()) fail("unexpected end");
    JsonValue v;
    const char c = t_[i_];
    if (c == '{') {
      ++i_;
      v.kind = JsonValue::object;
      if (eat('}')) return v;
      do {
        ws();
        std::string k = string_lit();
        expect(':');
        v.obj[k] = value();
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++i_;
      v.kind = JsonValue::array;
      if (eat(']')) return v;
      do v.arr.push_back(value());
      while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.kind = JsonValue::string;
      v.str = string_lit();
    } else if (word("true")) {
      v.kind = JsonValue::boolean;
      v.b = true;
    } else if (word("false")) {
      v.kind = JsonValue::boolean;
    } else if (word("null")) {
      v.kind = JsonValue::null;
    } else {
      number(v);
    }
    return v;
  }
  std::string string_lit() {
    if (i_ >= t_.size() || t_[i_] != '"') fail("expected a string");
    ++i_;
    std::string s;
    while (i_ < t_.size() && t_[i_] != '"') {
      char c = t_[i_++];
      if (c == '\\') {
        if (i_ >= t_.size()) fail("bad escape");
        const char e = t_[i_++];
        switch (e) {
          case 'n': c = '\n'; break;
          case 't': c = '\t'; break;
          case 'r': c = '\r'; break;
          case 'b': c = '\b'; break;
          case 'f': c = '\f'; break;
          case 'u': {
            if (i_ + 4 > t_.size()) fail("bad \\u escape");
            const unsigned cp = static_cast<unsigned>(std::strtoul(t_.substr(i_, 4).c_str(), nullptr, 16));
            i_ += 4;
            if (cp < 0x80) {
              c = static_cast<char>(cp);
            } else if (cp < 0x800) {
              s.push_back(static_cast<char>(0xC0 | (cp >> 6)));
              c = static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              s.push_back(static_cast<char>(0xE0 | (cp >> 12)));
              s.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
              c = static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: c = e; break;  // \" \\ \/
        }
      }
      s.push_back(c);
    }
    if (i_ >= t_.size()) fail("unterminated string");
    ++i_;
    return s;
  }
  void number(JsonValue& v) {
    const std::size_t s = i_;
    if (i_ < t_.size() && (t_[i_] == '-' || t_[i_] == '+')) ++i_;
    bool frac = false;
    while (i_ < t_.size()) {
      const char c = t_[i_];
      if (c >= '0' && c <= '9') {
        ++i_;
      } else if (c == '.' || c == 'e' || c == 'E' || ((c == '-' || c == '+') && frac)) {
        frac = true;
        ++i_;
      } else {
        break;
      }
    }
    if (i_ == s) fail("unexpected character");
    const std::string lit = t_.substr(s, i_ - s);
    v.kind = JsonValue::number;
    v.num = std::strtod(lit.c_str(), nullptr);
    v.is_int = !frac;
    if (v.is_int) v.inum = std::strtoll(lit.c_str(), nullptr, 10);
  }
  const std::string& t_;
  std::size_t i_ = 0;
};

}  // namespace ooc
