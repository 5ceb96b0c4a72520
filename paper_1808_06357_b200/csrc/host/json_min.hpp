// Minimal JSON value/parser/dumper for lattice specs and solver configs.
// Objects keep keys sorted (std::map), so dump() matches the compact,
// key-sorted form the reference emits through nlohmann::json
// (e.g. {"Z":[[1,34]],"d":2,"n":[55],"r":1}, lattice.cpp:340-347).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace lattdse::json {

struct Value {
  enum Kind { Null, Bool, Int, Float, String, Array, Object } kind = Null;
  bool b = false;
  std::int64_t i = 0;
  double f = 0.0;
  std::string s;
  std::vector<Value> arr;
  std::map<std::string, Value> obj;

  static Value integer(std::int64_t v) { Value x; x.kind = Int; x.i = v; return x; }
  static Value number(double v) { Value x; x.kind = Float; x.f = v; return x; }
  static Value string(std::string v) { Value x; x.kind = String; x.s = std::move(v); return x; }
  static Value array() { Value x; x.kind = Array; return x; }
  static Value object() { Value x; x.kind = Object; return x; }

  bool has(const std::string& k) const { return kind == Object && obj.count(k) != 0; }
  const Value& at(const std::string& k) const;
  std::int64_t as_int() const;      // throws std::runtime_error on type mismatch
  double as_double() const;
  std::string dump() const;
};

/// Parse a JSON document; throws std::runtime_error with a position on error.
Value parse(const std::string& text);

}  // namespace lattdse::json
