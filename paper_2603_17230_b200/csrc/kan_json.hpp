// kan_json.hpp -- minimal JSON reader for the reference descriptor schema
// (io.hpp:357-386, cost.hpp:214-246): objects, arrays, numbers, strings,
// true/false/null.  Throws kan::FormatError on malformed input.
#pragma once
#include <cstdlib>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace kan {

struct FormatError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Json {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  double num = 0.0;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;

  bool has(const std::string& k) const { return kind == Object && obj.count(k) != 0; }
  const Json& at(const std::string& k) const {
    if (kind != Object) throw FormatError("descriptor: expected an object");
    auto it = obj.find(k);
    if (it == obj.end()) throw FormatError("descriptor: missing key '" + k + "'");
    return it->second;
  }
  const Json& at(size_t i) const {
    if (kind != Array || i >= arr.size()) throw FormatError("descriptor: bad array index");
    return arr[i];
  }
  double number() const {
    if (kind != Number) throw FormatError("descriptor: expected a number");
    return num;
  }
  int integer() const {
    const double v = number();
    if (v != static_cast<double>(static_cast<int>(v)))
      throw FormatError("descriptor: expected an integer");
    return static_cast<int>(v);
  }
  const std::string& string() const {
    if (kind != String) throw FormatError("descriptor: expected a string");
    return str;
  }
  int value_int(const std::string& k, int dflt) const { return has(k) ? at(k).integer() : dflt; }

  static Json parse(const std::string& text) {
    size_t pos = 0;
    Json j = parse_value(text, pos);
    skip_ws(text, pos);
    if (pos != text.size()) throw FormatError("descriptor: trailing characters");
    return j;
  }

 private:
  static void skip_ws(const std::string& s, size_t& p) {
    while (p < s.size() && (s[p] == ' ' || s[p] == '\n' || s[p] == '\t' || s[p] == '\r')) ++p;
  }
  static Json parse_value(const std::string& s, size_t& p) {
    skip_ws(s, p);
    if (p >= s.size()) throw FormatError("descriptor: unexpected end of input");
    const char c = s[p];
    Json j;
    if (c == '{') {
      j.kind = Object;
      ++p;
      skip_ws(s, p);
      if (p < s.size() && s[p] == '}') {
        ++p;
        return j;
      }
      for (;;) {
        skip_ws(s, p);
        Json key = parse_value(s, p);
        if (key.kind != String) throw FormatError("descriptor: object key must be a string");
        skip_ws(s, p);
        if (p >= s.size() || s[p] != ':') throw FormatError("descriptor: expected ':'");
        ++p;
        j.obj[key.str] = parse_value(s, p);
        skip_ws(s, p);
        if (p < s.size() && s[p] == ',') {
          ++p;
          continue;
        }
        if (p < s.size() && s[p] == '}') {
          ++p;
          return j;
        }
        throw FormatError("descriptor: expected ',' or '}'");
      }
    }
    if (c == '[') {
      j.kind = Array;
      ++p;
      skip_ws(s, p);
      if (p < s.size() && s[p] == ']') {
        ++p;
        return j;
      }
      for (;;) {
        j.arr.push_back(parse_value(s, p));
        skip_ws(s, p);
        if (p < s.size() && s[p] == ',') {
          ++p;
          continue;
        }
        if (p < s.size() && s[p] == ']') {
          ++p;
          return j;
        }
        throw FormatError("descriptor: expected ',' or ']'");
      }
    }
    if (c == '"') {
      j.kind = String;
      ++p;
      while (p < s.size() && s[p] != '"') {
        if (s[p] == '\\') {
          ++p;
          if (p >= s.size()) break;
          const char e = s[p];
          j.str += (e == 'n') ? '\n' : (e == 't') ? '\t' : e;
        } else {
          j.str += s[p];
        }
        ++p;
      }
      if (p >= s.size()) throw FormatError("descriptor: unterminated string");
      ++p;
      return j;
    }
    if (s.compare(p, 4, "true") == 0) {
      j.kind = Bool;
      j.b = true;
      p += 4;
      return j;
    }
    if (s.compare(p, 5, "false") == 0) {
      j.kind = Bool;
      p += 5;
      return j;
    }
    if (s.compare(p, 4, "null") == 0) {
      p += 4;
      return j;
    }
    const char* begin = s.c_str() + p;
    char* end = nullptr;
    j.num = std::strtod(begin, &end);
    if (end == begin) throw FormatError("descriptor: invalid JSON value");
    j.kind = Number;
    p += static_cast<size_t>(end - begin);
    return j;
  }
};

}  // namespace kan
