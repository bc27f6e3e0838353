// Minimal streaming JSON writer (plan dumps, reports, audit rows).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

namespace ooc {

class JsonWriter {
 public:
  JsonWriter& begin_object() {
    sep();
    out_ += '{';
    first_.push_back(true);
    return *this;
  }
  JsonWriter& end_object() {
    out_ += '}';
    first_.pop_back();
    return *this;
  }
  JsonWriter& begin_array() {
    sep();
    out_ += '[';
    first_.push_back(true);
    return *this;
  }
  JsonWriter& end_array() {
    out_ += ']';
    first_.pop_back();
    return *this;
  }
  JsonWriter& key(const std::string& k) {
    sep();
    quote(k);
    out_ += ':';
    after_key_ = true;
    return *this;
  }
  JsonWriter& value(const std::string& s) {
    sep();
    quote(s);
    return *this;
  }
  JsonWriter& value(const char* s) { return value(std::string(s)); }
  JsonWriter& value(bool b) {
    sep();
    out_ += b ? "true" : "false";
    return *this;
  }
  JsonWriter& value(int v) { return value(static_cast<long long>(v)); }
  JsonWriter& value(long v) { return value(static_cast<long long>(v)); }
  JsonWriter& value(long long v) {
    sep();
    out_ += std::to_string(v);
    return *this;
  }
  JsonWriter& value(double v) {
    sep();
    if (!std::isfinite(v)) {
      out_ += "null";
      return *this;
    }
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    out_ += buf;
    return *this;
  }
  const std::string& str() const { return out_; }

 private:
  void sep() {
    if (after_key_) {
      after_key_ = false;
      return;
    }
    if (!first_.empty()) {
      if (!first_.back()) out_ += ',';
      first_.back() = false;
    }
  }
  void quote(const std::string& s) {
    out_ += '"';
    for (char c : s) {
      if (c == '"' || c == '\\') {
        out_ += '\\';
        out_ += c;
      } else if (static_cast<unsigned char>(c) < 0x20) {
        char b[8];
        std::snprintf(b, sizeof b, "\\u%04x", c);
        out_ += b;
      } else {
        out_ += c;
      }
    }
    out_ += '"';
  }
  std::string out_;
  std::vector<bool> first_;
  bool after_key_ = false;
};

}  // namespace ooc
