// Device-resident corpus for the exhaustive retrieval scan (host/retrieval.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "../kernels/launch.h"
#include "common.hpp"

namespace srh {

struct Comm;

class Corpus {
 public:
  // Reference Corpus (retrieval.hpp:21-33) in columnar form: embeddings
  // [n x d_emb], features [n x n_feat] (feature_names order), doc ids [n].
  Corpus(const float* emb, const float* feat, const int64_t* ids, long long n, int d_emb,
         int n_feat, int device);
  ~Corpus();
  Corpus(const Corpus&) = delete;
  Corpus& operator=(const Corpus&) = delete;

  // exhaustive_topk: keep = filter_candidates mask (null = every doc).
  // Returns min(k, #candidates) entries, written to device memory.
  int topk(const float* query, int d_query, double w0, const double* w, int n_w,
           const uint8_t* keep, int k, srk::TopkEntry* dev_out);
  int topk_host(const float* query, int d_query, double w0, const double* w, int n_w,
                const uint8_t* keep, int k, int64_t* ids_out, double* scores_out);
  // This rank's corpus is a shard (global doc ids); one NCCL all-gather of
  // k entries per rank + the same comparator merge = the single-device result.
  int topk_sharded(Comm* c, const float* query, int d_query, double w0, const double* w, int n_w,
                   const uint8_t* keep, int k, int64_t* ids_out, double* scores_out);
  long long last_candidates() const { return last_candidates_; }
  float last_scan_ms() const { return last_scan_ms_; }  // fp32 pass of the last call
  cudaStream_t stream() const { return stream_; }
  long long size() const { return n_; }

 private:
  long long prepare(const float* query, int d_query, double w0, const double* w, int n_w,
                    const uint8_t* keep, int k, srk::RetrievalScan& a);
  int device_;
  long long n_;
  int d_, f_;
  cudaStream_t stream_ = nullptr;
  float* emb_ = nullptr;
  float* feat_ = nullptr;
  int64_t* ids_ = nullptr;
  uint8_t* keep_ = nullptr;
  double* vec_ = nullptr;
  int32_t* counters_ = nullptr;
  int32_t* cand_ = nullptr;
  int grid_ = 0, cand_cap_ = 0;
  std::vector<double> fmax_;
  long long last_candidates_ = 0;
  float last_scan_ms_ = 0.f;
  cudaEvent_t ev_[2] = {nullptr, nullptr};
  template <typename T>
  struct Buf {
    T* ptr = nullptr;
    size_t cap = 0;
    ~Buf() {
      if (ptr) cudaFree(ptr);
    }
    void ensure(size_t n) {
      if (n <= cap) return;
      if (ptr) cudaFree(ptr);
      ptr = nullptr;
      SR_CUDA_CHECK(cudaMalloc(&ptr, n * sizeof(T)));
      cap = n;
    }
  };
  template <typename T>
  struct Pinned {  // page-locked host staging: small copies stay asynchronous
    T* ptr = nullptr;
    size_t cap = 0;
    ~Pinned() {
      if (ptr) cudaFreeHost(ptr);
    }
    void ensure(size_t n) {
      if (n <= cap) return;
      if (ptr) cudaFreeHost(ptr);
      ptr = nullptr;
      SR_CUDA_CHECK(cudaMallocHost(&ptr, n * sizeof(T)));
      cap = n;
    }
  };
  Pinned<float> h32_;
  Pinned<double> h64_;
  Pinned<int32_t> hcnt_;
  Pinned<srk::TopkEntry> hout_;
  Buf<srk::TopkEntry> entries_, select_, out_, gathered_, merged_;
  Buf<uint8_t> sort_;
  static constexpr int kScanMaxK = 512;  // the fp32 pass keeps <= 2048 candidates per CTA
};

}  // namespace srh
