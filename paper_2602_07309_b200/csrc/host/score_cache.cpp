#include "score_cache.hpp"

#include <algorithm>
#include <cctype>
#include <map>

#include "common.hpp"

namespace srh {

std::string canonical_query(const std::string& text,
                            const std::vector<std::pair<std::string, std::string>>& filters) {
  std::string out;
  out.reserve(text.size());
  bool gap = false;  // a whitespace run seen after some output
  for (const char ch : text) {
    const auto c = static_cast<unsigned char>(ch);
    if (std::isspace(c)) {
      gap = !out.empty();
      continue;
    }
    if (gap) out.push_back(' ');
    gap = false;
    out.push_back(static_cast<char>(std::tolower(c)));
  }
  std::map<std::string, std::vector<std::string>> by_attr;  // byte order of attr
  for (const auto& f : filters) by_attr[f.first].push_back(f.second);
  for (auto& [attr, values] : by_attr) {
    std::sort(values.begin(), values.end());
    out += '|';
    out += attr;
    out += '=';
    for (size_t i = 0; i < values.size(); ++i) {
      if (i) out += ',';
      out += values[i];
    }
  }
  return out;
}

uint64_t fnv1a64(const char* data, size_t len) {
  // The reference's offset basis is 1469598103934665603 (midtier.cpp:47), one
  // digit short of the published FNV-1a basis 14695981039346656037; signatures
  // must match the reference's, so the same constant is used here.
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < len; ++i) {
    h ^= static_cast<unsigned char>(data[i]);
    h *= 0x100000001b3ull;  // FNV prime
  }
  return h;
}

size_t CacheKeyHash::operator()(const CacheKey& k) const {
  auto mix = [](uint64_t h, uint64_t v) { return h ^ (v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2)); };
  uint64_t h = fnv1a64(k.searcher_id);
  h = mix(h, k.query_signature);
  h = mix(h, static_cast<uint64_t>(k.entity_id));
  h = mix(h, fnv1a64(k.model_version));
  return static_cast<size_t>(h);
}

ScoreCache::ScoreCache(size_t capacity) : capacity_(capacity) {
  if (capacity_ == 0) fail(SR_PARAMETER, "cache capacity must be >= 1");
}

bool ScoreCache::get(const CacheKey& key, double* out, int n) {
  std::lock_guard<std::mutex> lock(mu_);
  const auto it = index_.find(key);
  if (it == index_.end()) return false;
  const auto& v = it->second->scores;
  if (static_cast<int>(v.size()) != n)
    fail(SR_ALIGNMENT, "cached score row has " + std::to_string(v.size()) + " tasks, expected " +
                           std::to_string(n));
  std::copy(v.begin(), v.end(), out);
  lru_.splice(lru_.begin(), lru_, it->second);
  return true;
}

void ScoreCache::put(const CacheKey& key, const double* scores, int n) {
  std::lock_guard<std::mutex> lock(mu_);
  const auto it = index_.find(key);
  if (it != index_.end()) {
    const auto& v = it->second->scores;
    if (static_cast<int>(v.size()) != n || !std::equal(v.begin(), v.end(), scores))
      fail(SR_CONSISTENCY,
           "conflicting scores for one cache key; scores must be deterministic per (key, model "
           "version)");
    lru_.splice(lru_.begin(), lru_, it->second);
    return;
  }
  lru_.push_front({key, std::vector<double>(scores, scores + n)});
  index_[key] = lru_.begin();
  if (lru_.size() > capacity_) {
    index_.erase(lru_.back().key);
    lru_.pop_back();
  }
}

size_t ScoreCache::size() const {
  std::lock_guard<std::mutex> lock(mu_);
  return lru_.size();
}

}  // namespace srh
