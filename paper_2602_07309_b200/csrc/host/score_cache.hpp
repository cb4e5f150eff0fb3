// Deterministic score cache in front of the device scorer.
//
// Same contract as the reference's mid-tier cache (midtier.hpp / midtier.cpp:
// 14-100): entries keyed by (searcher id, query signature, entity id, model
// version), LRU over whole entries, a hit refreshes recency, a miss changes
// nothing, and putting different scores under an existing key is a
// Consistency error (scores are deterministic per key and model version --
// the device path is bit-reproducible across batch shapes, so this holds for
// it too). The value is the engine's score row (relevance + task heads in
// config order) instead of a std::map<std::string, double>; equality is
// per-double ==, as the map comparison.
#pragma once

#include <cstddef>
#include <cstdint>
#include <list>
#include <mutex>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

namespace srh {

// midtier.cpp:14-44: lowercase, whitespace runs -> one space, trimmed; then
// "|attr=v1,v2" per attribute in byte order of attr, values sorted. `filters`
// holds (attr, value) pairs; repeated attrs collect their values.
std::string canonical_query(const std::string& text,
                            const std::vector<std::pair<std::string, std::string>>& filters);
// midtier.cpp:46-53 (FNV-1a 64-bit prime; the reference's offset basis).
uint64_t fnv1a64(const char* data, size_t len);
inline uint64_t fnv1a64(const std::string& s) { return fnv1a64(s.data(), s.size()); }

struct CacheKey {
  std::string searcher_id;
  uint64_t query_signature = 0;
  int64_t entity_id = 0;
  std::string model_version;
  bool operator==(const CacheKey& o) const {
    return query_signature == o.query_signature && entity_id == o.entity_id &&
           searcher_id == o.searcher_id && model_version == o.model_version;
  }
};

struct CacheKeyHash {  // midtier.cpp:55-62
  size_t operator()(const CacheKey& k) const;
};

class ScoreCache {
 public:
  explicit ScoreCache(size_t capacity);  // SR_PARAMETER when 0 (midtier.cpp:64-68)

  // Copies the cached row (n values) into out and refreshes recency.
  bool get(const CacheKey& key, double* out, int n);
  void put(const CacheKey& key, const double* scores, int n);
  size_t size() const;
  size_t capacity() const { return capacity_; }

 private:
  struct Entry {
    CacheKey key;
    std::vector<double> scores;
  };
  size_t capacity_;
  mutable std::mutex mu_;
  std::list<Entry> lru_;  // front = most recent
  std::unordered_map<CacheKey, std::list<Entry>::iterator, CacheKeyHash> index_;
};

}  // namespace srh
