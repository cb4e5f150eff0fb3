#include "h2d.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.hpp"

namespace srh {

CopyPool::CopyPool(int n_threads) {
  for (int i = 1; i < n_threads; ++i) threads_.emplace_back(&CopyPool::work, this, i);
}

CopyPool::~CopyPool() {
  {
    std::lock_guard<std::mutex> lock(mu_);
    stop_ = true;
  }
  go_.notify_all();
  for (auto& t : threads_) t.join();
}

void CopyPool::part(int id, int parts) {
  // 4 KB-aligned slices so neighbouring threads do not share pages
  const size_t per = ((bytes_ + parts - 1) / parts + 4095) & ~size_t(4095);
  const size_t b = std::min(bytes_, per * id), e = std::min(bytes_, b + per);
  if (e > b) std::memcpy(dst_ + b, src_ + b, e - b);
}

void CopyPool::work(int id) {
  uint64_t seen = 0;
  for (;;) {
    {
      std::unique_lock<std::mutex> lock(mu_);
      go_.wait(lock, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
    }
    part(id, static_cast<int>(threads_.size()) + 1);
    {
      std::lock_guard<std::mutex> lock(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
}

void CopyPool::copy(void* dst, const void* src, size_t bytes) {
  if (threads_.empty() || bytes < (size_t(1) << 20)) {
    std::memcpy(dst, src, bytes);
    return;
  }
  {
    std::lock_guard<std::mutex> lock(mu_);
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    bytes_ = bytes;
    pending_ = static_cast<int>(threads_.size());
    ++gen_;
  }
  go_.notify_all();
  part(0, static_cast<int>(threads_.size()) + 1);
  std::unique_lock<std::mutex> lock(mu_);
  done_.wait(lock, [&] { return pending_ == 0; });
}

void StagedUpload::init() {
  SR_CUDA_CHECK(cudaGetDevice(&device_));
  int n = static_cast<int>(std::thread::hardware_concurrency());
  if (const char* v = std::getenv("SRK_H2D_THREADS")) n = std::atoi(v);
  pool_ = new CopyPool(std::max(1, std::min(n, 8)));
  for (int i = 0; i < kBufs; ++i) {
    SR_CUDA_CHECK(cudaMallocHost(&stage_[i], kChunk));
    SR_CUDA_CHECK(cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming));
  }
  ready_ = true;
}

StagedUpload::~StagedUpload() {
  if (!ready_) return;
  for (int i = 0; i < kBufs; ++i) {
    if (busy_[i]) cudaEventSynchronize(ev_[i]);
    cudaEventDestroy(ev_[i]);
    cudaFreeHost(stage_[i]);
  }
  delete pool_;
}

void StagedUpload::upload(void* dst, const void* src, size_t bytes, cudaStream_t stream) {
  if (bytes == 0) return;
  cudaPointerAttributes a{};
  const bool pinned = cudaPointerGetAttributes(&a, src) == cudaSuccess &&
                      (a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged);
  cudaGetLastError();  // clear a "not registered" status from the query
  static const bool staged = [] {
    const char* v = std::getenv("SRK_H2D_STAGED");
    return v == nullptr || std::atoi(v) != 0;
  }();
  if (pinned || !staged || bytes < (size_t(2) << 20)) {
    // (a small pageable copy is staged by the driver before the call returns)
    SR_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream));
    return;
  }
  if (!ready_) init();
  int i = 0;
  for (size_t off = 0; off < bytes; off += kChunk, i ^= 1) {
    const size_t n = std::min(kChunk, bytes - off);
    if (busy_[i]) SR_CUDA_CHECK(cudaEventSynchronize(ev_[i]));  // its DMA has drained
    pool_->copy(stage_[i], static_cast<const char*>(src) + off, n);
    SR_CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(dst) + off, stage_[i], n,
                                  cudaMemcpyHostToDevice, stream));
    SR_CUDA_CHECK(cudaEventRecord(ev_[i], stream));
    busy_[i] = true;
  }
}

}  // namespace srh
