// Text-side helpers around the scorer: the pointwise prompt split that turns
// (system, query context, document) into the shared prefix and one item
// (prompt.cpp:14-38, prompt.hpp:17-25), and the /score response body
// (score_result_to_json, service.cpp:380-391).
#include "prompt.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "common.hpp"

namespace srh {

namespace {
constexpr const char kPromptSuffix[] = "\nRelevant (Yes/No): ";  // prompt.hpp:23

std::vector<int32_t> bytes_to_tokens(const std::string& text, int max_seq) {  // tokenizer.cpp:10-20
  if (static_cast<long>(text.size()) > max_seq)
    fail(SR_LENGTH_OVERFLOW, "text of " + std::to_string(text.size()) +
                                 " bytes exceeds max_seq " + std::to_string(max_seq));
  std::vector<int32_t> t(text.size());
  for (size_t k = 0; k < text.size(); ++k) t[k] = static_cast<unsigned char>(text[k]);
  return t;
}
}  // namespace

PromptParts build_prompt(std::string_view system, std::string_view query_context,
                         std::string_view document, int max_seq) {
  std::string prefix;
  prefix.reserve(system.size() + query_context.size());
  prefix.append(system).append(query_context);
  std::string item;
  item.reserve(document.size() + sizeof(kPromptSuffix));
  item.append(document).append(kPromptSuffix);
  const size_t total = prefix.size() + item.size();
  // same checks, same order, same messages as prompt.cpp:25-33
  if (static_cast<long>(total) > max_seq)
    fail(SR_LENGTH_OVERFLOW, "prompt of " + std::to_string(total) + " tokens exceeds max_seq " +
                                 std::to_string(max_seq));
  if (prefix.empty())
    fail(SR_SPEC_VIOLATION, "prompt prefix (system + query context) must be non-empty");
  return {bytes_to_tokens(prefix, max_seq), bytes_to_tokens(item, max_seq)};
}

// ----------------------------------------------------------- JSON writer
// The reference serialises with nlohmann::json (3.11) dump(): objects are
// std::map-ordered (keys sorted bytewise), no whitespace, strings escaped with
// \" \\ \b \f \n \r \t and \u00xx (lower-case hex) for the other control
// bytes, UTF-8 validated; doubles are printed with Grisu2 (Loitsch, "Printing
// Floating-Point Numbers Quickly and Accurately with Integers", PLDI 2010:
// digits of the scaled upper boundary, cut as soon as the remainder lies
// inside the rounding interval, last digit nudged toward the value), laid
// out like printf %g with fixed notation for decimal point positions in
// (-4, 15] ("0.5", "15007744.0", "0.0001", "1e-05", "1.5e+20"), "-0.0" for
// negative zero, null for non-finite values. Grisu2 is not always shortest
// (about 0.4% of doubles above 1e14 get a longer or different digit string
// than a shortest-round-trip printer), so the reference's bytes need the
// same algorithm, not std::to_chars.
namespace {

struct Fp {  // f * 2^e
  uint64_t f;
  int e;
};

// 64 x 64 -> upper 64 bits, rounded half up on bit 63 of the 96-bit middle
// (the 32-bit partial-product formulation of the algorithm's "multiply").
Fp fp_mul(Fp a, Fp b) {
  const unsigned __int128 p = static_cast<unsigned __int128>(a.f) * b.f;
  const unsigned __int128 mid = (p >> 32) + (static_cast<unsigned __int128>(1) << 31);
  return {static_cast<uint64_t>(mid >> 32), a.e + b.e + 64};
}

Fp fp_normalize(Fp x) {
  const int lz = __builtin_clzll(x.f);
  return {x.f << lz, x.e - lz};
}

// Correctly rounded 64-bit significands of 10^k, k = -300, -292, ..., 324
// (generated with exact rational arithmetic).
struct Pow10 {
  uint64_t f;
  int e;
  int k;
};
constexpr Pow10 kPow10[] = {
    {0xAB70FE17C79AC6CAULL, -1060, -300}, {0xFF77B1FCBEBCDC4FULL, -1034, -292}, {0xBE5691EF416BD60CULL, -1007, -284},
    {0x8DD01FAD907FFC3CULL, -980, -276}, {0xD3515C2831559A83ULL, -954, -268}, {0x9D71AC8FADA6C9B5ULL, -927, -260},
    {0xEA9C227723EE8BCBULL, -901, -252}, {0xAECC49914078536DULL, -874, -244}, {0x823C12795DB6CE57ULL, -847, -236},
    {0xC21094364DFB5637ULL, -821, -228}, {0x9096EA6F3848984FULL, -794, -220}, {0xD77485CB25823AC7ULL, -768, -212},
    {0xA086CFCD97BF97F4ULL, -741, -204}, {0xEF340A98172AACE5ULL, -715, -196}, {0xB23867FB2A35B28EULL, -688, -188},
    {0x84C8D4DFD2C63F3BULL, -661, -180}, {0xC5DD44271AD3CDBAULL, -635, -172}, {0x936B9FCEBB25C996ULL, -608, -164},
    {0xDBAC6C247D62A584ULL, -582, -156}, {0xA3AB66580D5FDAF6ULL, -555, -148}, {0xF3E2F893DEC3F126ULL, -529, -140},
    {0xB5B5ADA8AAFF80B8ULL, -502, -132}, {0x87625F056C7C4A8BULL, -475, -124}, {0xC9BCFF6034C13053ULL, -449, -116},
    {0x964E858C91BA2655ULL, -422, -108}, {0xDFF9772470297EBDULL, -396, -100}, {0xA6DFBD9FB8E5B88FULL, -369, -92},
    {0xF8A95FCF88747D94ULL, -343, -84}, {0xB94470938FA89BCFULL, -316, -76}, {0x8A08F0F8BF0F156BULL, -289, -68},
    {0xCDB02555653131B6ULL, -263, -60}, {0x993FE2C6D07B7FACULL, -236, -52}, {0xE45C10C42A2B3B06ULL, -210, -44},
    {0xAA242499697392D3ULL, -183, -36}, {0xFD87B5F28300CA0EULL, -157, -28}, {0xBCE5086492111AEBULL, -130, -20},
    {0x8CBCCC096F5088CCULL, -103, -12}, {0xD1B71758E219652CULL, -77, -4}, {0x9C40000000000000ULL, -50, 4},
    {0xE8D4A51000000000ULL, -24, 12}, {0xAD78EBC5AC620000ULL, 3, 20}, {0x813F3978F8940984ULL, 30, 28},
    {0xC097CE7BC90715B3ULL, 56, 36}, {0x8F7E32CE7BEA5C70ULL, 83, 44}, {0xD5D238A4ABE98068ULL, 109, 52},
    {0x9F4F2726179A2245ULL, 136, 60}, {0xED63A231D4C4FB27ULL, 162, 68}, {0xB0DE65388CC8ADA8ULL, 189, 76},
    {0x83C7088E1AAB65DBULL, 216, 84}, {0xC45D1DF942711D9AULL, 242, 92}, {0x924D692CA61BE758ULL, 269, 100},
    {0xDA01EE641A708DEAULL, 295, 108}, {0xA26DA3999AEF774AULL, 322, 116}, {0xF209787BB47D6B85ULL, 348, 124},
    {0xB454E4A179DD1877ULL, 375, 132}, {0x865B86925B9BC5C2ULL, 402, 140}, {0xC83553C5C8965D3DULL, 428, 148},
    {0x952AB45CFA97A0B3ULL, 455, 156}, {0xDE469FBD99A05FE3ULL, 481, 164}, {0xA59BC234DB398C25ULL, 508, 172},
    {0xF6C69A72A3989F5CULL, 534, 180}, {0xB7DCBF5354E9BECEULL, 561, 188}, {0x88FCF317F22241E2ULL, 588, 196},
    {0xCC20CE9BD35C78A5ULL, 614, 204}, {0x98165AF37B2153DFULL, 641, 212}, {0xE2A0B5DC971F303AULL, 667, 220},
    {0xA8D9D1535CE3B396ULL, 694, 228}, {0xFB9B7CD9A4A7443CULL, 720, 236}, {0xBB764C4CA7A44410ULL, 747, 244},
    {0x8BAB8EEFB6409C1AULL, 774, 252}, {0xD01FEF10A657842CULL, 800, 260}, {0x9B10A4E5E9913129ULL, 827, 268},
    {0xE7109BFBA19C0C9DULL, 853, 276}, {0xAC2820D9623BF429ULL, 880, 284}, {0x80444B5E7AA7CF85ULL, 907, 292},
    {0xBF21E44003ACDD2DULL, 933, 300}, {0x8E679C2F5E44FF8FULL, 960, 308}, {0xD433179D9C8CB841ULL, 986, 316},
    {0x9E19DB92B4E31BA9ULL, 1013, 324},
};
constexpr int kPow10MinK = -300, kPow10Step = 8;
constexpr int kAlpha = -60;  // target window [alpha, gamma] for the scaled exponent

// Digits of v (finite, > 0): digits * 10^dec_exp.
void grisu2(double v, char* digits, int& len, int& dec_exp) {
  uint64_t bits;
  std::memcpy(&bits, &v, sizeof(bits));
  const uint64_t E = bits >> 52, F = bits & ((uint64_t{1} << 52) - 1);
  const Fp w = E == 0 ? Fp{F, 1 - 1075} : Fp{F | (uint64_t{1} << 52), static_cast<int>(E) - 1075};
  // rounding interval: halfway to the neighbours (the lower one is twice as
  // close when v is a power of two above the smallest normal)
  const Fp hi = fp_normalize({2 * w.f + 1, w.e - 1});
  Fp lo = (F == 0 && E > 1) ? Fp{4 * w.f - 1, w.e - 2} : Fp{2 * w.f - 1, w.e - 1};
  lo = {lo.f << (lo.e - hi.e), hi.e};
  const Fp wn = fp_normalize(w);
  // cached power c = 10^k putting hi's scaled exponent into [alpha, gamma]
  const int t = kAlpha - hi.e - 1;
  const int kk = (t * 78913) / (1 << 18) + (t > 0 ? 1 : 0);  // ceil(t log10 2)
  const Pow10& c = kPow10[(kk - kPow10MinK + kPow10Step - 1) / kPow10Step];
  const Fp sw = fp_mul(wn, {c.f, c.e});
  const Fp up = {fp_mul(hi, {c.f, c.e}).f - 1, sw.e};  // shrink by one unit each side:
  const Fp dn = {fp_mul(lo, {c.f, c.e}).f + 1, sw.e};  // every cut stays inside
  dec_exp = -c.k;
  uint64_t delta = up.f - dn.f;  // width of the safe interval
  uint64_t dist = up.f - sw.f;   // distance from the top to the scaled value
  const int sh = -up.e;
  const uint64_t one = uint64_t{1} << sh;
  uint32_t ip = static_cast<uint32_t>(up.f >> sh);  // integral part (< 2^32)
  uint64_t fr = up.f & (one - 1);                   // fractional part
  auto nudge = [&](uint64_t rest, uint64_t ten) {   // move the last digit toward v
    while (rest < dist && delta - rest >= ten &&
           (rest + ten < dist || dist - rest > rest + ten - dist)) {
      --digits[len - 1];
      rest += ten;
    }
  };
  len = 0;
  uint32_t p10 = 1;
  int n = 1;
  while (n < 10 && ip >= p10 * 10u) {
    p10 *= 10;
    ++n;
  }
  for (; n > 0; --n, p10 /= 10) {
    digits[len++] = static_cast<char>('0' + ip / p10);
    ip %= p10;
    const uint64_t rest = (static_cast<uint64_t>(ip) << sh) + fr;
    if (rest <= delta) {
      dec_exp += n - 1;
      nudge(rest, static_cast<uint64_t>(p10) << sh);
      return;
    }
  }
  for (int m = 1;; ++m) {
    fr *= 10;
    digits[len++] = static_cast<char>('0' + (fr >> sh));
    fr &= one - 1;
    delta *= 10;
    dist *= 10;
    if (fr <= delta) {
      dec_exp -= m;
      nudge(fr, one);
      return;
    }
  }
}

}  // namespace

void json_number(std::string& out, double v) {
  if (!std::isfinite(v)) {
    out += "null";
    return;
  }
  if (std::signbit(v)) {
    out.push_back('-');
    v = -v;
  }
  if (v == 0.0) {
    out += "0.0";
    return;
  }
  char buf[32];
  int k = 0, dec_exp = 0;
  grisu2(v, buf, k, dec_exp);
  const std::string digits(buf, static_cast<size_t>(k));
  const int n = k + dec_exp;  // position of the decimal point relative to the digits
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) {
    out += digits;
    out.append(static_cast<size_t>(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= kMaxExp) {
    out.append(digits, 0, static_cast<size_t>(n));
    out.push_back('.');
    out.append(digits, static_cast<size_t>(n), std::string::npos);
  } else if (kMinExp < n && n <= 0) {
    out += "0.";
    out.append(static_cast<size_t>(-n), '0');
    out += digits;
  } else {
    out.push_back(digits[0]);
    if (k > 1) {
      out.push_back('.');
      out.append(digits, 1, std::string::npos);
    }
    const int e = n - 1;
    char eb[8];
    std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
    out += eb;
  }
}

void json_string(std::string& out, std::string_view s) {
  out.push_back('"');
  for (size_t i = 0; i < s.size(); ++i) {
    const auto c = static_cast<unsigned char>(s[i]);
    switch (c) {
      case '"': out += "\\\""; continue;
      case '\\': out += "\\\\"; continue;
      case '\b': out += "\\b"; continue;
      case '\f': out += "\\f"; continue;
      case '\n': out += "\\n"; continue;
      case '\r': out += "\\r"; continue;
      case '\t': out += "\\t"; continue;
      default: break;
    }
    if (c < 0x20) {
      char buf[8];
      std::snprintf(buf, sizeof(buf), "\\u%04x", c);
      out += buf;
      continue;
    }
    if (c < 0x80) {
      out.push_back(static_cast<char>(c));
      continue;
    }
    // multi-byte UTF-8 sequence: validate, copy verbatim
    int len = c >= 0xF0 && c <= 0xF4 ? 4 : c >= 0xE0 ? 3 : c >= 0xC2 && c < 0xE0 ? 2 : 0;
    if (len == 0 || i + len > s.size())
      fail(SR_PAYLOAD_INVALID, "invalid UTF-8 byte at index " + std::to_string(i));
    const auto b1 = static_cast<unsigned char>(s[i + 1]);
    bool ok = (b1 & 0xC0) == 0x80;
    if (c == 0xE0) ok = ok && b1 >= 0xA0;
    if (c == 0xED) ok = ok && b1 < 0xA0;
    if (c == 0xF0) ok = ok && b1 >= 0x90;
    if (c == 0xF4) ok = ok && b1 < 0x90;
    for (int j = 2; j < len; ++j) ok = ok && (static_cast<unsigned char>(s[i + j]) & 0xC0) == 0x80;
    if (!ok) fail(SR_PAYLOAD_INVALID, "invalid UTF-8 byte at index " + std::to_string(i));
    out.append(s.substr(i, static_cast<size_t>(len)));
    i += static_cast<size_t>(len) - 1;
  }
  out.push_back('"');
}

std::string score_result_json(std::string_view request_id, int n_items,
                              const char* const* item_ids, int n_tasks,
                              const char* const* task_names, const double* scores,
                              double attention_units, double linear_units) {
  // task columns in name order (ItemScores::tasks is a std::map)
  std::vector<int> order(static_cast<size_t>(n_tasks));
  for (int t = 0; t < n_tasks; ++t) order[t] = t;
  std::sort(order.begin(), order.end(),
            [&](int a, int b) { return std::strcmp(task_names[a], task_names[b]) < 0; });
  for (int t = 1; t < n_tasks; ++t)
    if (std::strcmp(task_names[order[t - 1]], task_names[order[t]]) == 0)
      fail(SR_SPEC_VIOLATION, std::string("duplicate task name: ") + task_names[order[t]]);
  std::string out;
  out.reserve(96 + static_cast<size_t>(n_items) * (32 + 28 * n_tasks));
  out += "{\"flops\":{\"attention\":";
  json_number(out, attention_units);
  out += ",\"linear\":";
  json_number(out, linear_units);
  out += "},\"request_id\":";
  json_string(out, request_id);
  out += ",\"scores\":[";
  for (int i = 0; i < n_items; ++i) {
    if (i) out.push_back(',');
    out += "{\"id\":";
    json_string(out, item_ids[i] ? item_ids[i] : "");
    out += ",\"tasks\":{";
    for (int j = 0; j < n_tasks; ++j) {
      if (j) out.push_back(',');
      json_string(out, task_names[order[j]]);
      out.push_back(':');
      json_number(out, scores[static_cast<size_t>(i) * n_tasks + order[j]]);
    }
    out += "}}";
  }
  out += "]}";
  return out;
}

}  // namespace srh
