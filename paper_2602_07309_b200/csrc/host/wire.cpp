// Native /score wire parser: see wire.hpp.
#include "wire.hpp"

#include <cstring>

namespace srh {

namespace {

struct Scanner {
  const char* s;
  int64_t n;
  int64_t i = 0;

  [[noreturn]] void bad(const std::string& what) const {
    fail(SR_PAYLOAD_INVALID, "request body is not JSON: " + what + " at byte " + std::to_string(i));
  }
  void ws() {
    while (i < n && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) ++i;
  }
  char peek() {
    ws();
    if (i >= n) bad("unexpected end of input");
    return s[i];
  }
  void expect(char c) {
    if (peek() != c) bad(std::string("expected '") + c + "'");
    ++i;
  }
  // String span [b, e) of the raw (escaped) contents; sets esc when a
  // backslash occurs.
  void string_span(int64_t& b, int64_t& e, bool& esc) {
    expect('"');
    b = i;
    esc = false;
    for (;;) {
      const void* q = std::memchr(s + i, '"', static_cast<size_t>(n - i));
      if (q == nullptr) bad("unterminated string");
      const int64_t j = static_cast<const char*>(q) - s;
      // count backslashes right before the quote: odd -> escaped quote
      int64_t k = j;
      while (k > b && s[k - 1] == '\\') --k;
      if (std::memchr(s + i, '\\', static_cast<size_t>(j - i)) != nullptr) esc = true;
      if (((j - k) & 1) == 0) {
        e = j;
        i = j + 1;
        return;
      }
      i = j + 1;
    }
  }
  static void put_utf8(std::string& out, uint32_t cp) {
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
  uint32_t hex4(int64_t at) {
    if (at + 4 > n) bad("bad \\u escape");
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = s[at + k];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
      else bad("bad \\u escape");
    }
    return v;
  }
  std::string unescape(int64_t b, int64_t e) {
    std::string out;
    out.reserve(static_cast<size_t>(e - b));
    for (int64_t k = b; k < e; ++k) {
      const char c = s[k];
      if (c != '\\') {
        out.push_back(c);
        continue;
      }
      if (++k >= e) bad("bad escape");
      switch (s[k]) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          uint32_t cp = hex4(k + 1);
          k += 4;
          if (cp >= 0xD800 && cp < 0xDC00 && k + 6 < e && s[k + 1] == '\\' && s[k + 2] == 'u') {
            const uint32_t lo = hex4(k + 3);
            if (lo >= 0xDC00 && lo < 0xE000) {
              cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
              k += 6;
            }
          }
          put_utf8(out, cp);
          break;
        }
        default: bad("bad escape");
      }
    }
    return out;
  }
  std::string string_value() {
    int64_t b, e;
    bool esc;
    string_span(b, e, esc);
    return esc ? unescape(b, e) : std::string(s + b, static_cast<size_t>(e - b));
  }
  double number() {
    ws();
    const int64_t b = i;
    if (i < n && (s[i] == '-' || s[i] == '+')) ++i;
    while (i < n && ((s[i] >= '0' && s[i] <= '9') || s[i] == '.' || s[i] == 'e' || s[i] == 'E' ||
                     s[i] == '-' || s[i] == '+'))
      ++i;
    if (i == b) bad("expected a value");
    return std::strtod(std::string(s + b, static_cast<size_t>(i - b)).c_str(), nullptr);
  }
  void literal(const char* w) {
    const size_t L = std::strlen(w);
    if (i + static_cast<int64_t>(L) > n || std::strncmp(s + i, w, L) != 0) bad("bad literal");
    i += static_cast<int64_t>(L);
  }
  void skip_value() {
    const char c = peek();
    if (c == '"') {
      int64_t b, e;
      bool esc;
      string_span(b, e, esc);
    } else if (c == '{') {
      ++i;
      if (peek() == '}') {
        ++i;
        return;
      }
      for (;;) {
        int64_t b, e;
        bool esc;
        string_span(b, e, esc);
        expect(':');
        skip_value();
        if (peek() == ',') {
          ++i;
          continue;
        }
        expect('}');
        return;
      }
    } else if (c == '[') {
      ++i;
      if (peek() == ']') {
        ++i;
        return;
      }
      for (;;) {
        skip_value();
        if (peek() == ',') {
          ++i;
          continue;
        }
        expect(']');
        return;
      }
    } else if (c == 't') {
      literal("true");
    } else if (c == 'f') {
      literal("false");
    } else if (c == 'n') {
      literal("null");
    } else {
      number();
    }
  }
  bool boolean() {
    const char c = peek();
    if (c == 't') {
      literal("true");
      return true;
    }
    if (c == 'f') {
      literal("false");
      return false;
    }
    fail(SR_PAYLOAD_INVALID, "type error: expected a boolean");
  }
  std::vector<int32_t> int_array() {
    std::vector<int32_t> v;
    if (peek() != '[') fail(SR_PAYLOAD_INVALID, "type error: expected an array of integers");
    ++i;
    if (peek() == ']') {
      ++i;
      return v;
    }
    for (;;) {
      const double x = number();
      if (x != static_cast<double>(static_cast<int64_t>(x)))
        fail(SR_PAYLOAD_INVALID, "type error: expected an integer");
      v.push_back(static_cast<int32_t>(x));
      if (peek() == ',') {
        ++i;
        continue;
      }
      expect(']');
      return v;
    }
  }
  // Object members: calls f(key) positioned at the value; f consumes it.
  template <typename F>
  void object(F&& f) {
    expect('{');
    if (peek() == '}') {
      ++i;
      return;
    }
    for (;;) {
      const std::string key = string_value();
      expect(':');
      f(key);
      if (peek() == ',') {
        ++i;
        continue;
      }
      expect('}');
      return;
    }
  }
};

std::vector<int32_t> tokenize(const std::string& text, int max_seq) {  // tokenizer.cpp:10-20
  if (static_cast<long>(text.size()) > max_seq)
    fail(SR_LENGTH_OVERFLOW, "text of " + std::to_string(text.size()) +
                                 " bytes exceeds max_seq " + std::to_string(max_seq));
  std::vector<int32_t> t(text.size());
  for (size_t k = 0; k < text.size(); ++k) t[k] = static_cast<unsigned char>(text[k]);
  return t;
}

int32_t mode_from_name(const std::string& m) {  // engine.cpp:22-29
  if (m == "naive") return SR_MODE_NAIVE;
  if (m == "ibpc") return SR_MODE_IBPC;
  if (m == "multi_item" || m == "multi-item") return SR_MODE_MULTI_ITEM;
  if (m == "mixed") return SR_MODE_MIXED;
  fail(SR_PARAMETER, "unknown scoring mode: " + m);
}

}  // namespace

WireRequest parse_wire(const char* body, int64_t len, int max_seq) {
  WireRequest r;
  r.body = body;
  r.body_len = len;
  Scanner sc{body, len};
  bool have_prefix = false, have_items = false;
  std::string prefix_text;
  bool prefix_is_text = false;
  std::string mode = "ibpc";
  sc.object([&](const std::string& key) {
    if (key == "request_id") {
      r.request_id = sc.string_value();
    } else if (key == "prefix_tokens") {
      r.prefix = sc.int_array();
      have_prefix = true;
      prefix_is_text = false;
    } else if (key == "prefix_text" && !(have_prefix && !prefix_is_text)) {
      prefix_text = sc.string_value();
      have_prefix = true;
      prefix_is_text = true;
    } else if (key == "mode") {
      mode = sc.string_value();
    } else if (key == "latency_sensitive") {
      r.latency_sensitive = sc.boolean();
    } else if (key == "items") {
      if (sc.peek() != '[') {
        sc.skip_value();
        return;
      }
      have_items = true;
      ++sc.i;
      if (sc.peek() == ']') {
        ++sc.i;
        return;
      }
      for (;;) {
        WireRequest::Item it;
        int kind = -1;  // 0 tokens, 1 text, 2 b64 (reference precedence: tokens > text > b64)
        std::string text;
        int64_t bb = 0, be = 0;
        bool besc = false;
        sc.object([&](const std::string& k) {
          if (k == "id") {
            it.id = sc.string_value();
          } else if (k == "tokens") {
            it.tokens = sc.int_array();
            kind = 0;
          } else if (k == "text") {
            text = sc.string_value();
            if (kind != 0) kind = 1;
          } else if (k == "embedding_b64") {
            sc.string_span(bb, be, besc);
            if (kind < 0) kind = 2;
          } else {
            sc.skip_value();
          }
        });
        if (kind == 1) {
          it.tokens = tokenize(text, max_seq);
        } else if (kind == 2) {
          it.b64 = true;
          if (besc) {  // JSON escapes inside the payload (e.g. "\/"): unescape aside
            const std::string u = sc.unescape(bb, be);
            it.in_side = true;
            it.b64_begin = static_cast<int64_t>(r.side.size());
            r.side += u;
            it.b64_end = static_cast<int64_t>(r.side.size());
          } else {
            it.b64_begin = bb;
            it.b64_end = be;
          }
        } else if (kind < 0) {
          fail(SR_PAYLOAD_INVALID, "item needs text, tokens, or embedding_b64: " + it.id);
        }
        r.items.push_back(std::move(it));
        if (sc.peek() == ',') {
          ++sc.i;
          continue;
        }
        sc.expect(']');
        break;
      }
    } else {
      sc.skip_value();
    }
  });
  sc.ws();
  if (sc.i != len) sc.bad("trailing characters");
  if (!have_prefix) fail(SR_PAYLOAD_INVALID, "request needs prefix_text or prefix_tokens");
  if (prefix_is_text) r.prefix = tokenize(prefix_text, max_seq);
  r.mode = mode_from_name(mode);
  if (!have_items || r.items.empty())
    fail(SR_PAYLOAD_INVALID, "request needs a non-empty items[]");
  return r;
}

}  // namespace srh
