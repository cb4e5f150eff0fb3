// Minimal JSON value + parser/serializer for the SRNKWTS1 manifest
// (weights_io.cpp:56-96). Objects keep key order (needed only for dumping
// in the reference's key order); numbers are kept as text and converted on
// demand so 64-bit offsets survive.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "common.hpp"

namespace srh::json {

struct Value {
  enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
  bool b = false;
  std::string text;  // number text or string contents
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;

  const Value& at(const std::string& key) const {
    if (kind != Object) fail(SR_IO, "json: not an object (looking for '" + key + "')");
    for (const auto& kv : obj)
      if (kv.first == key) return kv.second;
    fail(SR_IO, "json: missing key '" + key + "'");
  }
  int64_t as_int() const {
    if (kind != Number) fail(SR_IO, "json: not a number");
    return std::stoll(text);
  }
  uint64_t as_uint() const {
    if (kind != Number) fail(SR_IO, "json: not a number");
    return std::stoull(text);
  }
  const std::string& as_str() const {
    if (kind != String) fail(SR_IO, "json: not a string");
    return text;
  }
};

Value parse(const std::string& s);

// Serializer helpers for the manifest writer.
std::string quote(const std::string& s);

}  // namespace srh::json
