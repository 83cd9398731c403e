// Minimal strict JSON reader for the fixed-schema files the planner reads
// (schedules, input lists). RFC 8259 grammar; numbers keep the integer /
// unsigned / float distinction a strict schema check needs; a repeated
// object key keeps its last value (as the reference's JSON library does).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace poas::json {

struct Value {
  enum class Type { null, boolean, integer, unsigned_integer, floating, string, array, object };
  Type type = Type::null;
  bool b = false;
  std::int64_t i = 0;
  std::uint64_t u = 0;
  double f = 0.0;
  std::string s;
  std::vector<Value> items;                     // array
  std::vector<std::pair<std::string, Value>> members;  // object, first-seen key order

  bool is_object() const { return type == Type::object; }
  bool is_array() const { return type == Type::array; }
  bool is_string() const { return type == Type::string; }
  bool is_integer() const { return type == Type::integer || type == Type::unsigned_integer; }
  bool is_number() const { return is_integer() || type == Type::floating; }

  const Value* get(const std::string& key) const;  // object lookup
  std::int64_t as_int64() const;                   // integer kinds (unsigned wraps)
  double as_double() const;                        // any number
  std::size_t size() const { return is_object() ? members.size() : items.size(); }
};

// Throws poas::Error(parse_failure, "<context>: <what>") on malformed text.
Value parse(const std::string& text, const std::string& context);

}  // namespace poas::json
