// Exhaustive filtered top-K retrieval scan: the stage
// upstream of the ranker. Reference: exhaustive_topk (retrieval.cpp:134-173),
// rar_score (:60-71), cosine (:44-58), TopK comparator (:99-103).
//
// B200 design: the scan is HBM-bound (D*4 + F*4 + 1 bytes per doc), but the
// reference scores in double, and fp64 throughput would bound a double scan
// ~100x below the HBM roofline. So:
//   pass 1  retrieval_scan_kernel: fp32 scores (FFMA, smem-staged coalesced
//           tiles), each CTA keeps every doc whose fp32 score is within 2 eps
//           of its running k-th best — eps a rigorous bound on |s32 - s64| —
//           which is a superset of the CTA's exact top-k;
//   pass 2  retrieval_refine_kernel: the few candidates rescored in double in
//           the reference's operation order (bit-identical scores);
//   pass 3  topk_select: exact top-k by (score desc, doc_id asc).
// A candidate overflow (pathological near-ties) is flagged and the host runs
// pass 2 over every doc instead.
#include <cuda_bf16.h>

#include <cub/device/device_radix_sort.cuh>

#include "launch.h"
#include "ptx.cuh"

namespace srk {

namespace {

constexpr int kScanThreads = 256;
constexpr int kCandCap = 2048;  // per-CTA candidate buffer
constexpr int kDimChunk = 32;

struct Cand {
  float s;
  int32_t idx;
};

__device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) { return a.s > b.s; }

// Bitonic sort of c[0..P) best-first (P power of two, padded with -inf).
__device__ void sort_cands(Cand* c, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const Cand a = c[lo], b = c[hi];
        if (asc ? cand_better(b, a) : cand_better(a, b)) {
          c[lo] = b;
          c[hi] = a;
        }
      }
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kScanThreads)
    retrieval_scan_kernel(RetrievalScan a, int32_t* __restrict__ g_cand, int g_cap,
                          int32_t* __restrict__ counters, long long docs_per_cta) {
  pdl_wait();
  // dynamic smem: candidates [kCandCap] | tile [256][33] | query [D]
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Cand* cand = reinterpret_cast<Cand*>(smem_raw);
  auto tile = reinterpret_cast<float(*)[kDimChunk + 1]>(smem_raw + kCandCap * sizeof(Cand));
  float* sq = reinterpret_cast<float*>(smem_raw + kCandCap * sizeof(Cand) +
                                       kScanThreads * (kDimChunk + 1) * sizeof(float));
  __shared__ int count;
  __shared__ float thr;
  __shared__ int overflow;
  const int t = threadIdx.x;
  const long long lo = static_cast<long long>(blockIdx.x) * docs_per_cta;
  const long long hi = min(a.n, lo + docs_per_cta);
  for (int i = t; i < a.D; i += kScanThreads) sq[i] = a.q32[i];
  if (t == 0) {
    count = 0;
    thr = -INFINITY;
    overflow = 0;
  }
  const float qn = static_cast<float>(a.q_norm);
  const float w0 = static_cast<float>(a.w0);

  // Keep the prefix of the sorted buffer within eps2 of the k-th best.
  auto compact = [&]() {
    __syncthreads();
    const int n = count;
    int P = 1;
    while (P < n) P <<= 1;
    for (int i = n + t; i < P; i += kScanThreads) cand[i] = Cand{-INFINITY, -1};
    sort_cands(cand, P);
    if (t == 0) {
      float th = thr;
      if (n >= a.k) th = fmaxf(th, cand[a.k - 1].s);
      thr = th;
      // entries are sorted: binary search the last one >= th - eps2
      int l = 0, r = n;
      while (l < r) {
        const int m = (l + r) >> 1;
        if (cand[m].s >= th - a.eps2) l = m + 1;
        else r = m;
      }
      if (l > kCandCap / 2) {  // too many near-ties to keep exactly
        l = kCandCap / 2;
        overflow = 1;
      }
      count = l;
    }
    __syncthreads();
  };

  __syncthreads();
  for (long long base = lo; base < hi; base += kScanThreads) {
    const long long doc = base + t;
    const int rows = static_cast<int>(min(static_cast<long long>(kScanThreads), hi - base));
    float dot = 0.f, nb = 0.f;
    for (int c0 = 0; c0 < a.D; c0 += kDimChunk) {
      const int cw = min(kDimChunk, a.D - c0);
      __syncthreads();
      // coalesced: consecutive threads read consecutive 16 B of doc rows
      if ((a.D & 3) == 0) {
        const int cw4 = cw >> 2;
        for (int e = t; e < rows * cw4; e += kScanThreads) {
          const int dd = e / cw4, ii = e - dd * cw4;
          const float4 v =
              __ldcs(reinterpret_cast<const float4*>(a.emb + (base + dd) * a.D + c0) + ii);
          tile[dd][4 * ii] = v.x;
          tile[dd][4 * ii + 1] = v.y;
          tile[dd][4 * ii + 2] = v.z;
          tile[dd][4 * ii + 3] = v.w;
        }
      } else {
        for (int e = t; e < rows * cw; e += kScanThreads) {
          const int dd = e / cw, ii = e - dd * cw;
          tile[dd][ii] = a.emb[(base + dd) * a.D + c0 + ii];
        }
      }
      __syncthreads();
      if (t < rows) {
#pragma unroll 8
        for (int ii = 0; ii < cw; ++ii) {
          const float v = tile[t][ii];
          dot = fmaf(sq[c0 + ii], v, dot);
          nb = fmaf(v, v, nb);
        }
      }
    }
    if (t < rows && (a.keep == nullptr || a.keep[doc] != 0)) {
      if (nb == 0.f) atomicOr(&counters[1], 1);
      float s = w0 * (dot / (qn * sqrtf(nb)));
      for (int f = 0; f < a.F; ++f) s = fmaf(a.w32[f], a.feat[doc * a.F + f], s);
      if (s >= thr - a.eps2) {
        const int slot = atomicAdd(&count, 1);
        cand[slot] = Cand{s, static_cast<int32_t>(doc)};
      }
    }
    __syncthreads();
    if (count > kCandCap - kScanThreads) compact();
  }
  if (count > 0) compact();
  __shared__ int gbase;
  if (t == 0) {
    gbase = count > 0 ? atomicAdd(&counters[0], count) : 0;
    if (overflow || gbase + count > g_cap) atomicOr(&counters[1], 2);
  }
  __syncthreads();
  if (gbase + count <= g_cap)
    for (int i = t; i < count; i += kScanThreads) g_cand[gbase + i] = cand[i].idx;
  pdl_trigger();
}


// TMA-streamed variant (D % 4 == 0): a tile of R docs is R*D*4 contiguous
// bytes, fetched by one 1D bulk copy into a 3-deep smem ring (no register
// staging, completion on an mbarrier). Thread t owns doc t of the tile and
// reads its row as float4s in a rotated order (chunk (j + t) mod D/4), which
// spreads each quarter-warp over distinct bank groups; the fp32 pass needs
// only the error bound, not the reference's summation order.
//
// Occupancy decides the bandwidth: the per-tile compute (two block barriers,
// the candidate test) is serial within a CTA, so more CTAs per SM beat deeper
// rings. Measured at 33.5M x d 32 (bench retrieval_xl): 1 CTA x 6 stages 0.51
// of HBM peak, 2 CTAs x 3 stages (2048 candidates) 0.82, 3 CTAs x 2 stages
// (1024 candidates) 0.98. The 3-CTA shape serves k <= 256; larger k (up to
// kCandCap / 4 = 512) takes the 2-CTA shape.
constexpr int kBulkTileBytes = 32768;
#ifndef SRK_SCAN_MIN_DOCS_PER_K
#define SRK_SCAN_MIN_DOCS_PER_K 16
#endif

template <int STAGES, int CAND>
struct ScanShape {
  static constexpr size_t smem(int D) {
    return STAGES * kBulkTileBytes + CAND * sizeof(Cand) +
           static_cast<size_t>((D + 3) & ~3) * sizeof(float) + 64;
  }
};

template <int kBulkStages, int kCandCap>
__global__ void __launch_bounds__(kScanThreads)
    retrieval_scan_bulk_kernel(RetrievalScan a, int32_t* __restrict__ g_cand, int g_cap,
                               int32_t* __restrict__ counters, long long docs_per_cta, int rows) {
  pdl_wait();
  // dynamic smem: ring [STAGES][32 KB] | candidates [CAND] | query [D] | barriers
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* ring = smem_raw;
  Cand* cand = reinterpret_cast<Cand*>(smem_raw + kBulkStages * kBulkTileBytes);
  float* sq = reinterpret_cast<float*>(cand + kCandCap);
  uint64_t* full = reinterpret_cast<uint64_t*>(sq + ((a.D + 3) & ~3));
  __shared__ int count;
  __shared__ float thr;
  __shared__ int overflow;
  const int t = threadIdx.x;
  const long long lo = static_cast<long long>(blockIdx.x) * docs_per_cta;
  const long long hi = min(a.n, lo + docs_per_cta);
  const int n_tiles = hi > lo ? static_cast<int>((hi - lo + rows - 1) / rows) : 0;
  const int D4 = a.D >> 2;
  for (int i = t; i < a.D; i += kScanThreads) sq[i] = a.q32[i];
  const uint64_t pol = policy_evict_first();  // streamed once
  auto issue = [&](int tile) {
    const long long base = lo + static_cast<long long>(tile) * rows;
    const int r = static_cast<int>(min(static_cast<long long>(rows), hi - base));
    const int st = tile % kBulkStages;
    mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(r) * a.D * 4);
    bulk_load_1d(ring + st * kBulkTileBytes, a.emb + base * a.D, static_cast<uint32_t>(r) * a.D * 4,
                 &full[st], pol);
  };
  if (t == 0) {
    count = 0;
    thr = -INFINITY;
    overflow = 0;
    for (int s = 0; s < kBulkStages; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
    for (int s = 0; s < kBulkStages && s < n_tiles; ++s) issue(s);
  }
  const float qn = static_cast<float>(a.q_norm);
  const float w0 = static_cast<float>(a.w0);

  auto compact = [&]() {
    __syncthreads();
    const int n = count;
    int P = 1;
    while (P < n) P <<= 1;
    for (int i = n + t; i < P; i += kScanThreads) cand[i] = Cand{-INFINITY, -1};
    sort_cands(cand, P);
    if (t == 0) {
      float th = thr;
      if (n >= a.k) th = fmaxf(th, cand[a.k - 1].s);
      thr = th;
      int l = 0, r = n;
      while (l < r) {
        const int m = (l + r) >> 1;
        if (cand[m].s >= th - a.eps2) l = m + 1;
        else r = m;
      }
      if (l > kCandCap / 2) {
        l = kCandCap / 2;
        overflow = 1;
      }
      count = l;
    }
    __syncthreads();
  };

  __syncthreads();
  for (int tile = 0; tile < n_tiles; ++tile) {
    const long long base = lo + static_cast<long long>(tile) * rows;
    const int r = static_cast<int>(min(static_cast<long long>(rows), hi - base));
    const int st = tile % kBulkStages;
    mbar_wait(&full[st], (tile / kBulkStages) & 1);
    float dot0 = 0.f, dot1 = 0.f, nb0 = 0.f, nb1 = 0.f;
    const long long doc = base + t;
    if (t < r) {
      const float4* row = reinterpret_cast<const float4*>(ring + st * kBulkTileBytes) + t * D4;
      int j = t % D4;
#pragma unroll 4
      for (int c = 0; c < D4; ++c) {
        const float4 v = row[j];
        const float4 qv = reinterpret_cast<const float4*>(sq)[j];
        dot0 = fmaf(qv.x, v.x, dot0);
        dot1 = fmaf(qv.y, v.y, dot1);
        dot0 = fmaf(qv.z, v.z, dot0);
        dot1 = fmaf(qv.w, v.w, dot1);
        nb0 = fmaf(v.x, v.x, nb0);
        nb1 = fmaf(v.y, v.y, nb1);
        nb0 = fmaf(v.z, v.z, nb0);
        nb1 = fmaf(v.w, v.w, nb1);
        j = j + 1 == D4 ? 0 : j + 1;
      }
    }
    __syncthreads();  // every thread is done with this stage
    if (t == 0 && tile + kBulkStages < n_tiles) issue(tile + kBulkStages);
    if (t < r && (a.keep == nullptr || a.keep[doc] != 0)) {
      const float dot = dot0 + dot1, nb = nb0 + nb1;
      if (nb == 0.f) atomicOr(&counters[1], 1);
      float s = w0 * (dot / (qn * sqrtf(nb)));
      for (int f = 0; f < a.F; ++f) s = fmaf(a.w32[f], a.feat[doc * a.F + f], s);
      if (s >= thr - a.eps2) {
        const int slot = atomicAdd(&count, 1);
        cand[slot] = Cand{s, static_cast<int32_t>(doc)};
      }
    }
    __syncthreads();
    if (count > kCandCap - kScanThreads) compact();
  }
  if (count > 0) compact();
  __shared__ int gbase;
  if (t == 0) {
    gbase = count > 0 ? atomicAdd(&counters[0], count) : 0;
    if (overflow || gbase + count > g_cap) atomicOr(&counters[1], 2);
  }
  __syncthreads();
  if (gbase + count <= g_cap)
    for (int i = t; i < count; i += kScanThreads) g_cand[gbase + i] = cand[i].idx;
  pdl_trigger();
}

// Exact rescoring in the reference's order: dot, na, nb accumulated in
// double over float products (exact), cos = dot / (sqrt(na) * sqrt(nb)),
// s = w0 * cos, s += w_i * f_i (retrieval.cpp:44-71). Round-to-nearest
// intrinsics keep nvcc from contracting into FMAs.
__global__ void retrieval_refine_kernel(RetrievalScan a, const int32_t* __restrict__ cand,
                                        long long n_cand, TopkEntry* __restrict__ out,
                                        int32_t* __restrict__ counters) {
  pdl_wait();
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_cand) return;
  const long long doc = cand != nullptr ? cand[i] : i;
  TopkEntry e;
  e.id = INT64_MAX;
  e.index = INT32_MAX;
  e.pad = 0;
  e.score = -INFINITY;
  if (a.keep == nullptr || a.keep[doc] != 0) {
    const float* row = a.emb + doc * a.D;
    double dot = 0.0, nb = 0.0;
    for (int j = 0; j < a.D; ++j) {
      const double b = static_cast<double>(row[j]);
      dot = __dadd_rn(dot, __dmul_rn(a.qd[j], b));
      nb = __dadd_rn(nb, __dmul_rn(b, b));
    }
    if (nb == 0.0) atomicOr(&counters[1], 1);
    double s = __dmul_rn(a.w0, __ddiv_rn(dot, __dmul_rn(a.q_norm, __dsqrt_rn(nb))));
    for (int f = 0; f < a.F; ++f)
      s = __dadd_rn(s, __dmul_rn(a.wd[f], static_cast<double>(a.feat[doc * a.F + f])));
    e.score = s;
    e.id = a.ids[doc];
    e.index = static_cast<int32_t>(doc);
  }
  out[i] = e;
  pdl_trigger();
}

__global__ void split_entries_kernel(const TopkEntry* __restrict__ e, long long n,
                                     int64_t* __restrict__ id_keys, double* __restrict__ score,
                                     int32_t* __restrict__ idx) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  id_keys[i] = e[i].id;
  score[i] = e[i].score;
  idx[i] = static_cast<int32_t>(i);
}

__global__ void gather_scores_kernel(const double* __restrict__ score,
                                     const int32_t* __restrict__ perm, long long n,
                                     double* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = score[perm[i]];
}

__global__ void gather_entries_kernel(const TopkEntry* __restrict__ e,
                                      const int32_t* __restrict__ perm, int k,
                                      TopkEntry* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) out[i] = e[perm[i]];
}

}  // namespace

size_t retrieval_sort_scratch(long long n) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<int64_t*>(nullptr),
                                  static_cast<int64_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                  static_cast<int32_t*>(nullptr), static_cast<int>(n));
  cub::DeviceRadixSort::SortPairsDescending(nullptr, b, static_cast<double*>(nullptr),
                                            static_cast<double*>(nullptr),
                                            static_cast<int32_t*>(nullptr),
                                            static_cast<int32_t*>(nullptr), static_cast<int>(n));
  // cub temp + id keys x2 + scores x2 + indices x2
  return (a > b ? a : b) + static_cast<size_t>(n) * (2 * 8 + 2 * 8 + 2 * 4) + 7 * 256;
}

cudaError_t retrieval_sort_topk(const TopkEntry* e, long long n, int k, void* scratch,
                                size_t scratch_bytes, TopkEntry* out, cudaStream_t stream) {
  if (n <= 0 || k <= 0) return cudaSuccess;
  const int nn = static_cast<int>(n);
  uint8_t* p = static_cast<uint8_t*>(scratch);
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += (bytes + 255) / 256 * 256;
    return r;
  };
  int64_t* id0 = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* id1 = reinterpret_cast<int64_t*>(take(n * 8));
  double* s0 = reinterpret_cast<double*>(take(n * 8));
  double* s1 = reinterpret_cast<double*>(take(n * 8));
  int32_t* i0 = reinterpret_cast<int32_t*>(take(n * 4));
  int32_t* i1 = reinterpret_cast<int32_t*>(take(n * 4));
  const size_t used = static_cast<size_t>(p - static_cast<uint8_t*>(scratch));
  if (used > scratch_bytes) return cudaErrorInvalidValue;
  size_t temp = scratch_bytes - used;
  const int th = 256;
  const unsigned blocks = static_cast<unsigned>((n + th - 1) / th);
  split_entries_kernel<<<blocks, th, 0, stream>>>(e, n, id0, s0, i0);
  // stable: ascending doc id first, then descending score (ties keep id order)
  cudaError_t err = cub::DeviceRadixSort::SortPairs(p, temp, id0, id1, i0, i1, nn, 0, 64, stream);
  if (err != cudaSuccess) return err;
  gather_scores_kernel<<<blocks, th, 0, stream>>>(s0, i1, n, s1);
  temp = scratch_bytes - used;
  err = cub::DeviceRadixSort::SortPairsDescending(p, temp, s1, s0, i1, i0, nn, 0, 64, stream);
  if (err != cudaSuccess) return err;
  const int kk = static_cast<int>(k < n ? k : n);
  gather_entries_kernel<<<(kk + th - 1) / th, th, 0, stream>>>(e, i0, kk, out);
  return cudaGetLastError();
}

cudaError_t retrieval_scan(const RetrievalScan& a, int32_t* cand, int cand_cap, int32_t* counters,
                           int grid, cudaStream_t stream) {
  if (a.n <= 0) return cudaSuccess;
  if (a.k <= 0 || a.k > kCandCap / 4 || a.D <= 0) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(counters, 0, 2 * sizeof(int32_t), stream);
  if (e != cudaSuccess) return e;
  // contiguous doc ranges, a multiple of the tile size
  if ((a.D & 3) == 0 && a.D <= 128) {
    // TMA-streamed scan: tiles of `rows` docs (<= 32 KB, <= one per thread)
    const int rows = min(kScanThreads, kBulkTileBytes / (a.D * 4));
    int dev = 0;
    cudaGetDevice(&dev);
    const bool small_k = a.k <= 256;
    const int per_sm = small_k ? 3 : 2;
    const int g2 = min(grid, per_sm * num_sms(dev));
    long long per = (a.n + g2 - 1) / g2;
    // each CTA keeps ~k candidates: small corpora get fewer, longer CTAs so
    // the exact rescoring does not see most of the corpus
    per = std::max<long long>(per, static_cast<long long>(SRK_SCAN_MIN_DOCS_PER_K) * a.k);
    per = (per + rows - 1) / rows * rows;
    const int blocks = static_cast<int>((a.n + per - 1) / per);
    auto go = [&](auto kern, size_t smem) {
      cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (r != cudaSuccess) return r;
      return launch_k(kern, dim3(blocks), dim3(kScanThreads), smem, stream, a, cand, cand_cap,
                      counters, per, rows);
    };
    if (small_k) return go(retrieval_scan_bulk_kernel<2, 1024>, ScanShape<2, 1024>::smem(a.D));
    return go(retrieval_scan_bulk_kernel<3, kCandCap>, ScanShape<3, kCandCap>::smem(a.D));
  }
  long long per = (a.n + grid - 1) / grid;
  per = (per + kScanThreads - 1) / kScanThreads * kScanThreads;
  const int blocks = static_cast<int>((a.n + per - 1) / per);
  const size_t smem = kCandCap * sizeof(Cand) + kScanThreads * (kDimChunk + 1) * sizeof(float) +
                      static_cast<size_t>(a.D) * sizeof(float);
  e = cudaFuncSetAttribute(retrieval_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  return launch_k(retrieval_scan_kernel, dim3(blocks), dim3(kScanThreads), smem, stream, a, cand,
                  cand_cap, counters, per);
}

cudaError_t retrieval_refine(const RetrievalScan& a, const int32_t* cand, long long n_cand,
                             TopkEntry* out, int32_t* counters, cudaStream_t stream) {
  if (n_cand <= 0) return cudaSuccess;
  const int threads = 256;
  return launch_k(retrieval_refine_kernel, dim3(static_cast<unsigned>((n_cand + threads - 1) / threads)),
                  dim3(threads), 0, stream, a, cand, n_cand, out, counters);
}

}  // namespace srk
