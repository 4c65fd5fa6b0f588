// tuckerplan (B200 engine) : a small JSON value for the on-disk formats of serialize.hpp.
// The reference uses nlohmann::json (a third-party header that is not part of its tree); this type covers what the
// formats and the command line need with the same observable conventions: objects keep their keys sorted, dump(2)
// indents by two spaces with one member per line, integers print exactly (u64 / i64), doubles print the shortest
// text that reads back to the same value, parse() returns a discarded value on malformed input instead of throwing.
#pragma once

#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "errors.hpp"

namespace tuckerplan {

class Json {
 public:
  enum class Type { null, boolean, uinteger, integer, real, string, array, object, discarded };
  using Array = std::vector<Json>;
  using Object = std::map<std::string, Json>;

  Json() = default;
  Json(std::nullptr_t) {}
  Json(bool b) : type_(Type::boolean), bool_(b) {}
  Json(int v) : type_(v < 0 ? Type::integer : Type::uinteger), int_(v), uint_(static_cast<std::uint64_t>(v)) {}
  Json(long v) : type_(v < 0 ? Type::integer : Type::uinteger), int_(v), uint_(static_cast<std::uint64_t>(v)) {}
  Json(long long v) : type_(v < 0 ? Type::integer : Type::uinteger), int_(v), uint_(static_cast<std::uint64_t>(v)) {}
  Json(unsigned v) : type_(Type::uinteger), uint_(v) {}
  Json(unsigned long v) : type_(Type::uinteger), uint_(v) {}
  Json(unsigned long long v) : type_(Type::uinteger), uint_(v) {}
  Json(double v) : type_(Type::real), real_(v) {}
  Json(const char* s) : type_(Type::string), string_(s) {}
  Json(std::string s) : type_(Type::string), string_(std::move(s)) {}
  template <class T>
  Json(const std::vector<T>& values) : type_(Type::array) {
    for (const T& v : values) array_.emplace_back(v);
  }

  static Json array() {
    Json j;
    j.type_ = Type::array;
    return j;
  }
  static Json object() {
    Json j;
    j.type_ = Type::object;
    return j;
  }
  static Json object(std::initializer_list<std::pair<const std::string, Json>> members) {
    Json j = object();
    for (const auto& kv : members) j.object_[kv.first] = kv.second;
    return j;
  }

  Type type() const { return type_; }
  bool is_discarded() const { return type_ == Type::discarded; }
  bool is_object() const { return type_ == Type::object; }
  bool is_array() const { return type_ == Type::array; }
  bool is_string() const { return type_ == Type::string; }
  bool is_number() const { return type_ == Type::uinteger || type_ == Type::integer || type_ == Type::real; }
  bool empty() const { return is_array() ? array_.empty() : is_object() ? object_.empty() : type_ == Type::null; }
  std::size_t size() const { return is_array() ? array_.size() : is_object() ? object_.size() : 0; }
  bool contains(const std::string& key) const { return is_object() && object_.count(key) != 0; }

  Json& operator[](const std::string& key) {
    if (type_ == Type::null) type_ = Type::object;
    if (!is_object()) fail(Errc::bad_argument, "JSON value is not an object");
    return object_[key];
  }
  const Json& at(const std::string& key) const {
    if (!is_object()) fail(Errc::bad_argument, "JSON value is not an object");
    const auto it = object_.find(key);
    if (it == object_.end()) fail(Errc::bad_argument, "JSON object lacks key " + key);
    return it->second;
  }
  const Json& at(std::size_t i) const {
    if (!is_array() || i >= array_.size()) fail(Errc::bad_argument, "JSON array index out of range");
    return array_[i];
  }
  void push_back(Json v) {
    if (type_ == Type::null) type_ = Type::array;
    if (!is_array()) fail(Errc::bad_argument, "JSON value is not an array");
    array_.push_back(std::move(v));
  }
  const Array& items() const { return array_; }
  const Object& members() const { return object_; }

  std::uint64_t as_u64() const {
    if (type_ == Type::uinteger) return uint_;
    if (type_ == Type::integer && int_ >= 0) return static_cast<std::uint64_t>(int_);
    fail(Errc::bad_argument, "JSON value is not a non-negative integer");
  }
  double as_double() const {
    if (type_ == Type::real) return real_;
    if (type_ == Type::uinteger) return static_cast<double>(uint_);
    if (type_ == Type::integer) return static_cast<double>(int_);
    fail(Errc::bad_argument, "JSON value is not a number");
  }
  bool as_bool() const {
    if (type_ != Type::boolean) fail(Errc::bad_argument, "JSON value is not a boolean");
    return bool_;
  }
  const std::string& as_string() const {
    if (type_ != Type::string) fail(Errc::bad_argument, "JSON value is not a string");
    return string_;
  }
  template <class T>
  std::vector<T> as_vector_u64() const {
    if (!is_array()) fail(Errc::bad_argument, "JSON value is not an array");
    std::vector<T> out;
    for (const Json& v : array_) out.push_back(static_cast<T>(v.as_u64()));
    return out;
  }

  // indent < 0: compact on one line; otherwise one member per line, `indent` spaces per level
  std::string dump(int indent = -1) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

  static Json parse(const std::string& text) {
    Parser p{text, 0};
    Json v = p.value();
    p.skip();
    if (p.bad || p.at != text.size()) {
      Json d;
      d.type_ = Type::discarded;
      return d;
    }
    return v;
  }

 private:
  Type type_ = Type::null;
  bool bool_ = false;
  std::int64_t int_ = 0;
  std::uint64_t uint_ = 0;
  double real_ = 0.0;
  std::string string_;
  Array array_;
  Object object_;

  static void write_string(std::string& out, const std::string& s) {
    out += '"';
    for (const char ch : s) {
      const unsigned char c = static_cast<unsigned char>(ch);
      switch (c) {
        case '"': out += "\\\""; break;
        case '\\': out += "\\\\"; break;
        case '\b': out += "\\b"; break;
        case '\f': out += "\\f"; break;
        case '\n': out += "\\n"; break;
        case '\r': out += "\\r"; break;
        case '\t': out += "\\t"; break;
        default:
          if (c < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof buf, "\\u%04x", c);
            out += buf;
          } else {
            out += ch;
          }
      }
    }
    out += '"';
  }

  static void write_real(std::string& out, double v) {
    if (!std::isfinite(v)) {
      out += "null";
      return;
    }
    char buf[40];
    const auto r = std::to_chars(buf, buf + sizeof buf, v);  // shortest round-trip text
    std::string text(buf, r.ptr);
    if (text.find_first_of(".eEn") == std::string::npos) text += ".0";
    out += text;
  }

  void write(std::string& out, int indent, int depth) const {
    const auto newline = [&](int d) {
      if (indent >= 0) {
        out += '\n';
        out.append(static_cast<std::size_t>(indent) * d, ' ');
      }
    };
    switch (type_) {
      case Type::null:
      case Type::discarded: out += "null"; break;
      case Type::boolean: out += bool_ ? "true" : "false"; break;
      case Type::uinteger: out += std::to_string(uint_); break;
      case Type::integer: out += std::to_string(int_); break;
      case Type::real: write_real(out, real_); break;
      case Type::string: write_string(out, string_); break;
      case Type::array:
        if (array_.empty()) {
          out += "[]";
          break;
        }
        out += '[';
        for (std::size_t i = 0; i < array_.size(); ++i) {
          if (i) out += ',';
          newline(depth + 1);
          array_[i].write(out, indent, depth + 1);
        }
        newline(depth);
        out += ']';
        break;
      case Type::object: {
        if (object_.empty()) {
          out += "{}";
          break;
        }
        out += '{';
        bool first = true;
        for (const auto& kv : object_) {
          if (!first) out += ',';
          first = false;
          newline(depth + 1);
          write_string(out, kv.first);
          out += indent >= 0 ? ": " : ":";
          kv.second.write(out, indent, depth + 1);
        }
        newline(depth);
        out += '}';
        break;
      }
    }
  }

  struct Parser {
    const std::string& text;
    std::size_t at;
    bool bad = false;
    int depth = 0;

    void skip() {
      while (at < text.size() && (text[at] == ' ' || text[at] == '\n' || text[at] == '\t' || text[at] == '\r')) ++at;
    }
    bool eat(char c) {
      skip();
      if (at < text.size() && text[at] == c) {
        ++at;
        return true;
      }
      return false;
    }
    Json fail_value() {
      bad = true;
      return Json();
    }
    bool literal(const char* word) {
      const std::size_t n = std::char_traits<char>::length(word);
      if (text.compare(at, n, word) != 0) return false;
      at += n;
      return true;
    }
    std::string string_body() {
      std::string out;
      while (at < text.size() && text[at] != '"') {
        char c = text[at++];
        if (static_cast<unsigned char>(c) < 0x20) {
          bad = true;
          return out;
        }
        if (c != '\\') {
          out += c;
          continue;
        }
        if (at >= text.size()) break;
        c = text[at++];
        switch (c) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (at + 4 > text.size()) {
              bad = true;
              return out;
            }
            unsigned code = 0;
            for (int i = 0; i < 4; ++i) {
              const char h = text[at++];
              code <<= 4;
              if (h >= '0' && h <= '9') code |= static_cast<unsigned>(h - '0');
              else if (h >= 'a' && h <= 'f') code |= static_cast<unsigned>(h - 'a' + 10);
              else if (h >= 'A' && h <= 'F') code |= static_cast<unsigned>(h - 'A' + 10);
              else bad = true;
            }
            if (code < 0x80) {
              out += static_cast<char>(code);
            } else if (code < 0x800) {
              out += static_cast<char>(0xC0 | (code >> 6));
              out += static_cast<char>(0x80 | (code & 0x3F));
            } else {
              out += static_cast<char>(0xE0 | (code >> 12));
              out += static_cast<char>(0x80 | ((code >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (code & 0x3F));
            }
            break;
          }
          default: bad = true; return out;
        }
      }
      if (at >= text.size()) {
        bad = true;
        return out;
      }
      ++at;  // closing quote
      return out;
    }
    Json number() {
      const std::size_t begin = at;
      if (at < text.size() && text[at] == '-') ++at;
      if (at >= text.size() || text[at] < '0' || text[at] > '9') return fail_value();
      if (text[at] == '0' && at + 1 < text.size() && text[at + 1] >= '0' && text[at + 1] <= '9') return fail_value();
      bool integral = true;
      while (at < text.size() && text[at] >= '0' && text[at] <= '9') ++at;
      if (at < text.size() && text[at] == '.') {
        integral = false;
        ++at;
        if (at >= text.size() || text[at] < '0' || text[at] > '9') return fail_value();
        while (at < text.size() && text[at] >= '0' && text[at] <= '9') ++at;
      }
      if (at < text.size() && (text[at] == 'e' || text[at] == 'E')) {
        integral = false;
        ++at;
        if (at < text.size() && (text[at] == '+' || text[at] == '-')) ++at;
        if (at >= text.size() || text[at] < '0' || text[at] > '9') return fail_value();
        while (at < text.size() && text[at] >= '0' && text[at] <= '9') ++at;
      }
      const char* first = text.data() + begin;
      const char* last = text.data() + at;
      if (integral) {
        if (*first == '-') {
          std::int64_t v = 0;
          const auto r = std::from_chars(first, last, v);
          if (r.ec == std::errc() && r.ptr == last) return Json(static_cast<long long>(v));
        } else {
          std::uint64_t v = 0;
          const auto r = std::from_chars(first, last, v);
          if (r.ec == std::errc() && r.ptr == last) return Json(static_cast<unsigned long long>(v));
        }
      }
      double v = 0.0;
      const auto r = std::from_chars(first, last, v);
      if (r.ec != std::errc() || r.ptr != last) return fail_value();
      return Json(v);
    }
    Json value() {
      if (++depth > 200) return fail_value();
      skip();
      Json out;
      if (at >= text.size()) {
        out = fail_value();
      } else if (text[at] == '{') {
        ++at;
        out = Json::object();
        if (!eat('}')) {
          do {
            skip();
            if (at >= text.size() || text[at] != '"') {
              out = fail_value();
              break;
            }
            ++at;
            const std::string key = string_body();
            if (bad || !eat(':')) {
              out = fail_value();
              break;
            }
            out.object_[key] = value();
            if (bad) break;
          } while (eat(','));
          if (!bad && !eat('}')) out = fail_value();
        }
      } else if (text[at] == '[') {
        ++at;
        out = Json::array();
        if (!eat(']')) {
          do {
            out.array_.push_back(value());
            if (bad) break;
          } while (eat(','));
          if (!bad && !eat(']')) out = fail_value();
        }
      } else if (text[at] == '"') {
        ++at;
        out = Json(string_body());
      } else if (literal("true")) {
        out = Json(true);
      } else if (literal("false")) {
        out = Json(false);
      } else if (literal("null")) {
        out = Json();
      } else {
        out = number();
      }
      --depth;
      return out;
    }
  };
};

using json = Json;

}  // namespace tuckerplan
