#include "json_lite.hpp"

#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "poas/error.hpp"

namespace poas::json {

const Value* Value::get(const std::string& key) const {
  for (const auto& m : members)
    if (m.first == key) return &m.second;
  return nullptr;
}

std::int64_t Value::as_int64() const {
  if (type == Type::unsigned_integer) return static_cast<std::int64_t>(u);
  if (type == Type::integer) return i;
  if (type == Type::floating) return static_cast<std::int64_t>(f);
  return 0;
}

double Value::as_double() const {
  switch (type) {
    case Type::integer: return static_cast<double>(i);
    case Type::unsigned_integer: return static_cast<double>(u);
    case Type::floating: return f;
    default: return 0.0;
  }
}

namespace {

class Reader {
 public:
  Reader(const std::string& t, const std::string& ctx) : t_(t), ctx_(ctx) {}

  Value document() {
    ws();
    Value v = value(0);
    ws();
    if (p_ != t_.size()) error("unexpected trailing characters");
    return v;
  }

 private:
  [[noreturn]] void error(const std::string& what) const {
    fail(errc::parse_failure, ctx_ + ": parse error at byte " + std::to_string(p_) + ": " + what);
  }

  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r'))
      ++p_;
  }

  bool eat(char c) {
    if (p_ < t_.size() && t_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }

  void literal(const char* word) {
    const std::size_t n = std::strlen(word);
    if (t_.compare(p_, n, word) != 0) error(std::string("expected '") + word + "'");
    p_ += n;
  }

  Value value(int depth) {
    if (depth > 512) error("nesting too deep");
    if (p_ >= t_.size()) error("unexpected end of input");
    Value v;
    switch (t_[p_]) {
      case '{': return object(depth);
      case '[': return array(depth);
      case '"':
        v.type = Value::Type::string;
        v.s = string();
        return v;
      case 't':
        literal("true");
        v.type = Value::Type::boolean;
        v.b = true;
        return v;
      case 'f':
        literal("false");
        v.type = Value::Type::boolean;
        return v;
      case 'n':
        literal("null");
        return v;
      default: return number();
    }
  }

  Value object(int depth) {
    Value v;
    v.type = Value::Type::object;
    ++p_;  // '{'
    ws();
    if (eat('}')) return v;
    for (;;) {
      ws();
      if (p_ >= t_.size() || t_[p_] != '"') error("expected object key");
      std::string key = string();
      ws();
      if (!eat(':')) error("expected ':'");
      ws();
      Value item = value(depth + 1);
      bool replaced = false;
      for (auto& m : v.members)
        if (m.first == key) {
          m.second = std::move(item);
          replaced = true;
          break;
        }
      if (!replaced) v.members.emplace_back(std::move(key), std::move(item));
      ws();
      if (eat('}')) return v;
      if (!eat(',')) error("expected ',' or '}'");
    }
  }

  Value array(int depth) {
    Value v;
    v.type = Value::Type::array;
    ++p_;  // '['
    ws();
    if (eat(']')) return v;
    for (;;) {
      ws();
      v.items.push_back(value(depth + 1));
      ws();
      if (eat(']')) return v;
      if (!eat(',')) error("expected ',' or ']'");
    }
  }

  static void put_utf8(std::string& out, std::uint32_t cp) {
    if (cp < 0x80) {
      out.push_back(static_cast<char>(cp));
    } else if (cp < 0x800) {
      out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
      out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else {
      out.push_back(static_cast<char>(0xF0 | (cp >> 18)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    }
  }

  std::uint32_t hex4() {
    if (p_ + 4 > t_.size()) error("truncated \\u escape");
    std::uint32_t v = 0;
    for (int j = 0; j < 4; ++j) {
      const char c = t_[p_++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<std::uint32_t>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<std::uint32_t>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<std::uint32_t>(c - 'A' + 10);
      else error("bad \\u escape");
    }
    return v;
  }

  std::string string() {
    ++p_;  // opening quote
    std::string out;
    for (;;) {
      if (p_ >= t_.size()) error("unterminated string");
      const unsigned char c = static_cast<unsigned char>(t_[p_++]);
      if (c == '"') return out;
      if (c < 0x20) error("control character in string");
      if (c != '\\') {
        out.push_back(static_cast<char>(c));
        continue;
      }
      if (p_ >= t_.size()) error("unterminated escape");
      const char e = t_[p_++];
      switch (e) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          std::uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (!(eat('\\') && eat('u'))) error("unpaired surrogate");
            const std::uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) error("bad low surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            error("unpaired surrogate");
          }
          put_utf8(out, cp);
          break;
        }
        default: error("bad escape");
      }
    }
  }

  Value number() {
    const std::size_t start = p_;
    const bool neg = eat('-');
    if (p_ >= t_.size() || !std::isdigit(static_cast<unsigned char>(t_[p_]))) error("bad number");
    if (t_[p_] == '0') {
      ++p_;
    } else {
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
    }
    bool is_float = false;
    if (p_ < t_.size() && t_[p_] == '.') {
      is_float = true;
      ++p_;
      if (p_ >= t_.size() || !std::isdigit(static_cast<unsigned char>(t_[p_])))
        error("bad fraction");
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      is_float = true;
      ++p_;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      if (p_ >= t_.size() || !std::isdigit(static_cast<unsigned char>(t_[p_])))
        error("bad exponent");
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
    }
    const std::string tok = t_.substr(start, p_ - start);
    Value v;
    if (!is_float) {
      errno = 0;
      char* end = nullptr;
      if (neg) {
        const long long x = std::strtoll(tok.c_str(), &end, 10);
        if (errno != ERANGE) {
          v.type = Value::Type::integer;
          v.i = x;
          return v;
        }
      } else {
        const unsigned long long x = std::strtoull(tok.c_str(), &end, 10);
        if (errno != ERANGE) {
          v.type = Value::Type::unsigned_integer;
          v.u = x;
          return v;
        }
      }
      // Out of integer range: stored as a float, like the reference's reader.
    }
    errno = 0;
    v.type = Value::Type::floating;
    v.f = std::strtod(tok.c_str(), nullptr);
    if (!std::isfinite(v.f)) error("number out of range");
    return v;
  }

  const std::string& t_;
  const std::string& ctx_;
  std::size_t p_ = 0;
};

}  // namespace

Value parse(const std::string& text, const std::string& context) {
  return Reader(text, context).document();
}

}  // namespace poas::json
