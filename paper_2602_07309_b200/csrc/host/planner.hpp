// Host planner: request validation, FLOP accounting, multi-item masks,
// batch planning, and packing of one or more scoring requests into the
// ragged row layout the device pass consumes.
//
// Reference behaviour mirrored here (engine.cpp):
//   flops / actual_flops            :30-88
//   require_token_mode              :51-61
//   build_multi_item_mask, pairs    :147-184
//   score_multi_item positions      :209-217 (prefix-relative, T_q + j)
//   score_mixed payload checks      :243-251
//   plan_batches                    :278-326
//   score_multi_item_chunked plan   :328-377
// All token modes (naive / ibpc / multi_item) compute the same function: the
// reference's own tests hold them equal (test_engine.cpp:140-187) and the
// survey measured them bit-identical. The device therefore runs one packed
// shared-prefix pass for every mode; the modes differ only in validation
// and in the FlopReport they return.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <new>
#include <vector>

#include <cuda_runtime.h>

#include "../kernels/launch.h"
#include "model.hpp"

namespace srh {

// Marker for mixed-mode rows that arrive as base64 text (Engine::score_b64).
inline const float kB64RowsTag = 0.f;
#define kB64Rows (&::srh::kB64RowsTag)
// Marker for mixed-mode rows produced on the device from compact per-item
// embeddings (Engine::score_emb: zero-pad or projection).
inline const float kEmbRowsTag = 0.f;
#define kEmbRows (&::srh::kEmbRowsTag)

sr_flop_report flops(int mode, int64_t t_q, int64_t t_i, int64_t n_items);

struct ItemView {
  int32_t length;  // tokens or soft rows
};

// Validates one request against the model (throws srh::Error with the
// reference's error category) and returns per-item lengths.
std::vector<int32_t> validate_request(const ModelConfig& cfg, const sr_request& req);

// FlopReport + kv_incremental_per_item as the reference reports them for
// this request's mode (including chunk re-payment for multi_item).
void report_for(const ModelConfig& cfg, const sr_request& req, const std::vector<int32_t>& lens,
                sr_flop_report* flops_out, double* kv_out);

// Page-locked host storage for the packed arrays, so their uploads are
// asynchronous DMA (no driver staging copy per array); plain heap memory
// when no device is present (host-only tests).
template <typename T>
struct PinnedAlloc {
  using value_type = T;
  PinnedAlloc() = default;
  template <typename U>
  PinnedAlloc(const PinnedAlloc<U>&) {}
  T* allocate(size_t n) {
    void* p = nullptr;
    if (cudaMallocHost(&p, n * sizeof(T)) != cudaSuccess) {
      cudaGetLastError();  // clear: fall back to pageable memory
      p = std::malloc(n * sizeof(T));
      if (p == nullptr) throw std::bad_alloc();
      std::lock_guard<std::mutex> lock(registry_mu());
      pageable_registry().push_back(p);
    }
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t) {
    {
      std::lock_guard<std::mutex> lock(registry_mu());
      auto& reg = pageable_registry();
      for (auto& q : reg)
        if (q == p) {
          q = reg.back();
          reg.pop_back();
          std::free(p);
          return;
        }
    }
    cudaFreeHost(p);
  }
  static std::vector<void*>& pageable_registry() {
    static std::vector<void*> r;
    return r;
  }
  static std::mutex& registry_mu() {
    static std::mutex m;
    return m;
  }
  bool operator==(const PinnedAlloc&) const { return true; }
  bool operator!=(const PinnedAlloc&) const { return false; }
};
template <typename T>
using pinned_vector = std::vector<T, PinnedAlloc<T>>;

struct PackedBatch {
  int32_t M = 0;                       // packed rows
  int32_t n_items = 0;                 // items over all requests
  int32_t max_seg_len = 0;             // longest request (items)
  pinned_vector<int32_t> row_src;      // token id, or -(1 + soft row index)
  pinned_vector<int32_t> row_pos;      // positional-embedding index
  pinned_vector<srk::RowSpan> spans;   // attention mask per row
  pinned_vector<srk::AttnTile> tiles;  // attention work tiles
  pinned_vector<int32_t> last_rows;    // per item: packed row scored
  pinned_vector<int64_t> ids;          // per item: doc id for the tie rule
  pinned_vector<int32_t> seg_off;      // per request: item offsets [n_req + 1]
  // mixed-mode rows [R x d]: not copied on the host — each request's item
  // rows are already contiguous (item_offsets index them in order), so the
  // engine copies them straight from the caller's buffer into HBM.
  struct SoftSrc {
    const float* rows;
    size_t n_rows;
  };
  std::vector<SoftSrc> soft_src;  // rows == kB64Rows: decoded on the device
  int32_t n_soft = 0;
};

// Packs requests back to back. Row layout for request q (base = first row):
//   prefix rows  base .. base+T_q-1 : pos j,       keys [base, r]          (causal)
//   item i rows  s_i .. s_i+L_i-1   : pos T_q + j, keys [base, base+T_q) U [s_i, r]
// `id_base` offsets default ids (index within the request) for sharding.
void pack_requests(const ModelConfig& cfg, const sr_request* reqs, int n_req,
                   const std::vector<std::vector<int32_t>>& lens, PackedBatch& out);

// The packed layout (row_pos, spans, tiles, last_rows, seg_off, M, n_items,
// n_soft) depends only on each request's (t_q, mode, item lengths):
// layout_signature writes that key; pack_sources refills what changes between
// requests of one layout (row_src token ids, ids, soft-row sources) into an
// `out` that pack_requests filled for the same signature.
void layout_signature(const sr_request* reqs, int n_req,
                      const std::vector<std::vector<int32_t>>& lens, std::vector<int32_t>& sig);
void pack_sources(const sr_request* reqs, int n_req,
                  const std::vector<std::vector<int32_t>>& lens, PackedBatch& out);

int64_t multi_item_pair_count(int32_t prefix_len, const int32_t* lens, int n);

struct BatchEntry {
  int32_t request_index, item_begin, item_end;
};
struct Batch {
  std::vector<BatchEntry> entries;
  int64_t token_count = 0;
};
std::vector<Batch> plan_batches(const std::vector<int32_t>& prefix_len,
                                const std::vector<std::vector<int32_t>>& item_len,
                                int64_t max_batch_tokens);

struct HostTopk {
  double score;
  int64_t id;
  int32_t index;
};
std::vector<HostTopk> topk_host(const double* scores, const int64_t* ids, int32_t n, int32_t k);

}  // namespace srh
