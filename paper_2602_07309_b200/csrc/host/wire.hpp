// Native /score wire parser (service.cpp:326-372, parse_score_request_json)
// for the B200 engine: one pass over the JSON body; embedding_b64 payloads
// are kept as spans into the caller's body (never copied into host strings)
// and decoded on the device (kernels/wire.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"

namespace srh {

struct WireRequest {
  const char* body = nullptr;  // caller-owned, must outlive the request
  int64_t body_len = 0;
  std::string request_id;
  std::vector<int32_t> prefix;
  int32_t mode = SR_MODE_IBPC;
  bool latency_sensitive = false;
  struct Item {
    std::string id;
    std::vector<int32_t> tokens;  // tokens / text items
    bool b64 = false;
    int64_t b64_begin = 0, b64_end = 0;  // span in body, or in `side` when escaped
    bool in_side = false;
  };
  std::vector<Item> items;
  std::string side;  // unescaped embedding_b64 payloads that contained JSON escapes
};

// Errors as the reference: SR_PAYLOAD_INVALID ("request body is not JSON: ...",
// "request needs prefix_text or prefix_tokens", "request needs a non-empty
// items[]", "item needs text, tokens, or embedding_b64: <id>"), SR_LENGTH_OVERFLOW
// for text longer than max_seq (tokenizer.cpp:10-20), SR_PARAMETER for an
// unknown mode name (engine.cpp:22-29).
WireRequest parse_wire(const char* body, int64_t len, int max_seq);

}  // namespace srh
