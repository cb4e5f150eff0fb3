// Host -> device uploads of caller-owned (pageable) buffers.
//
// A pageable cudaMemcpyAsync is staged by the driver through one thread at
// ~10 GB/s; the soft-row payloads of mixed-mode requests (C3: 33.5 MB per
// call) made that the largest part of the end-to-end time. StagedUpload
// copies chunks into two pinned staging buffers with a small thread pool
// (host memory bandwidth scales with threads) while the previous chunk's DMA
// runs, so the upload approaches the PCIe DMA rate. Page-locked sources go
// straight to DMA.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <mutex>
#include <thread>
#include <vector>

namespace srh {

class CopyPool {
 public:
  explicit CopyPool(int n_threads);
  ~CopyPool();
  CopyPool(const CopyPool&) = delete;
  CopyPool& operator=(const CopyPool&) = delete;
  // memcpy split across the pool (the caller copies one part); blocks.
  void copy(void* dst, const void* src, size_t bytes);

 private:
  void work(int id);
  void part(int id, int parts);
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable go_, done_;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
};

class StagedUpload {
 public:
  StagedUpload() = default;
  ~StagedUpload();
  StagedUpload(const StagedUpload&) = delete;
  StagedUpload& operator=(const StagedUpload&) = delete;
  // Enqueues dst <- src (bytes) on `stream`. Returns once src may be reused
  // by the caller (its bytes are in pinned staging or already on the device).
  void upload(void* dst, const void* src, size_t bytes, cudaStream_t stream);

 private:
  static constexpr int kBufs = 2;
  static constexpr size_t kChunk = size_t(8) << 20;
  void init();
  bool ready_ = false;
  int device_ = -1;
  CopyPool* pool_ = nullptr;
  char* stage_[kBufs] = {};
  cudaEvent_t ev_[kBufs] = {};
  bool busy_[kBufs] = {};
};

}  // namespace srh
