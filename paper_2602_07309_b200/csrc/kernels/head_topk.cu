// Fused final LayerNorm + last-token score head, and the exact top-k.
//
// Score head (model.cpp:294-352): only the last row of each item is read;
// LN_f (gain-only, eps 1e-5) is applied to that row, then the few columns the
// reference actually consumes are evaluated: w_vocab[:, yes], w_vocab[:, no]
// (vocab_logits, model.cpp:309-316, of which yes_no_probability reads two
// entries) and every task head column (multi_head_scores, model.cpp:318-343).
// Probabilities are computed in double exactly as the reference does:
//   relevance = stable logistic of (l_no - l_yes)     (model.cpp:294-307)
//   arity-1 head: stable logistic of z = h.w + b      (model.cpp:329-332)
//   arity>1 head: softmax probability of class 0      (model.cpp:333-339)
//
// Top-k (semrank_main.cpp:393-398, service.cpp:271-277, retrieval.cpp:99-173):
// order by score descending, ties by ascending doc id, then by input index
// (== std::stable_sort for duplicate ids). One CTA bitonic-sorts up to 4096
// candidates in shared memory; larger segments are cut into chunks whose
// per-chunk top-k are merged by a second pass.
#include <cuda_bf16.h>

#include <cstdint>

#include "launch.h"

namespace srk {

namespace {

constexpr float kLnEps = 1e-5f;

template <int NV>
__global__ void __launch_bounds__(256)
    score_head_kernel(const float* __restrict__ x, const int32_t* __restrict__ last_rows,
                      int n_items, int d, const float* __restrict__ gain,
                      const float* __restrict__ w_cols, const float* __restrict__ bias,
                      int n_cols, const int32_t* __restrict__ task_col,
                      const int32_t* __restrict__ task_arity, int n_tasks, int yes_col,
                      int no_col, double* __restrict__ scores, float* __restrict__ hidden_out) {
  pdl_wait();
  extern __shared__ float s_logits[];  // [8 warps][n_cols]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * 8 + warp;
  if (item >= n_items) return;
  float* logits = s_logits + warp * n_cols;
  const int d4 = d >> 2;
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<size_t>(last_rows[item]) * d);
  float4 v[NV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < d4) {
      v[i] = xr[c];
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  const float mean = s / static_cast<float>(d);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < d4) {
      const float a = v[i].x - mean, b = v[i].y - mean, e = v[i].z - mean, f = v[i].w - mean;
      q += (a * a + b * b) + (e * e + f * f);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffff, q, o);
  const float inv = 1.0f / sqrtf(q / static_cast<float>(d) + kLnEps);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < d4) {
      const float4 g = reinterpret_cast<const float4*>(gain)[c];
      v[i].x = (v[i].x - mean) * inv * g.x;
      v[i].y = (v[i].y - mean) * inv * g.y;
      v[i].z = (v[i].z - mean) * inv * g.z;
      v[i].w = (v[i].w - mean) * inv * g.w;
      if (hidden_out != nullptr)
        reinterpret_cast<float4*>(hidden_out + static_cast<size_t>(item) * d)[c] = v[i];
    }
  }
  for (int col = 0; col < n_cols; ++col) {
    const float4* w = reinterpret_cast<const float4*>(w_cols + static_cast<size_t>(col) * d);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + i * 32;
      if (c < d4) {
        const float4 ww = w[c];
        acc += (v[i].x * ww.x + v[i].y * ww.y) + (v[i].z * ww.z + v[i].w * ww.w);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffff, acc, o);
    if (lane == 0) logits[col] = acc + bias[col];
  }
  __syncwarp();
  // lane 0 -> relevance, lanes 1..n_tasks-1 -> heads
  const int n_out = n_tasks;  // includes relevance at column 0
  for (int t = lane; t < n_out; t += 32) {
    double p;
    if (t == 0) {
      const double diff = static_cast<double>(logits[no_col]) - static_cast<double>(logits[yes_col]);
      if (diff > 0) {
        const double e = exp(-diff);
        p = e / (1.0 + e);
      } else {
        p = 1.0 / (1.0 + exp(diff));
      }
    } else {
      const int c0 = task_col[t - 1], ar = task_arity[t - 1];
      if (ar == 1) {
        const double z = static_cast<double>(logits[c0]);
        p = z >= 0 ? 1.0 / (1.0 + exp(-z)) : exp(z) / (1.0 + exp(z));
      } else {
        double mx = static_cast<double>(logits[c0]);
        for (int j = 1; j < ar; ++j) mx = fmax(mx, static_cast<double>(logits[c0 + j]));
        double den = 0.0;
        for (int j = 0; j < ar; ++j) den += exp(static_cast<double>(logits[c0 + j]) - mx);
        p = exp(static_cast<double>(logits[c0]) - mx) / den;
      }
    }
    scores[static_cast<size_t>(item) * n_out + t] = p;
  }
}

template <int NV>
cudaError_t launch_head(const float* x, const int32_t* last_rows, int n_items, int d,
                        const float* gain, const float* w_cols, const float* bias, int n_cols,
                        const int32_t* task_col, const int32_t* task_arity, int n_tasks,
                        int yes_col, int no_col, double* scores, float* hidden_out,
                        cudaStream_t stream) {
  const size_t smem = static_cast<size_t>(8) * n_cols * sizeof(float);
  return launch_k(score_head_kernel<NV>, dim3((n_items + 7) / 8), dim3(256), smem, stream, x,
                  last_rows, n_items, d, gain, w_cols, bias, n_cols, task_col, task_arity, n_tasks,
                  yes_col, no_col, scores, hidden_out);
}

// ------------------------------------------------------------------ top-k
constexpr int kSortCap = 4096;
constexpr int kSortThreads = 1024;

__device__ __forceinline__ bool better(const TopkEntry& a, const TopkEntry& b) {
  if (a.score != b.score) return a.score > b.score;
  if (a.id != b.id) return a.id < b.id;
  return a.index < b.index;
}

__device__ __forceinline__ TopkEntry sentinel() {
  TopkEntry e;
  e.score = -INFINITY;
  e.id = INT64_MAX;
  e.index = INT32_MAX;
  e.pad = 0;
  return e;
}

// Bitonic sort of buf[0..P) into "best first" order. P is a power of two.
__device__ void bitonic_sort(TopkEntry* buf, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < P / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;  // "asc" == best-first segment
        TopkEntry a = buf[lo], b = buf[hi];
        const bool swap = asc ? better(b, a) : better(a, b);
        if (swap) {
          buf[lo] = b;
          buf[hi] = a;
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ int pow2_at_least(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Stage 1: block b sorts chunk b of a segment (from raw scores).
// chunk_seg / chunk_lo / chunk_hi computed on the fly from seg_off.
__global__ void __launch_bounds__(kSortThreads)
    topk_scores_kernel(const double* __restrict__ scores, int stride,
                       const int64_t* __restrict__ ids, const int32_t* __restrict__ seg_off,
                       int n_segments, int k, TopkEntry* __restrict__ out, int chunks_per_seg) {
  pdl_wait();
  extern __shared__ TopkEntry buf[];
  const int seg = blockIdx.x / chunks_per_seg;
  const int chunk = blockIdx.x % chunks_per_seg;
  if (seg >= n_segments) return;
  const int lo = seg_off[seg] + chunk * kSortCap;
  const int hi = min(seg_off[seg + 1], lo + kSortCap);
  const int n = hi > lo ? hi - lo : 0;
  TopkEntry* dst = out + static_cast<size_t>(blockIdx.x) * k;
  if (n == 0) {
    for (int j = threadIdx.x; j < k; j += blockDim.x) dst[j] = sentinel();
    return;
  }
  const int P = pow2_at_least(n);
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    if (i < n) {
      const int idx = lo + i;
      TopkEntry e;
      e.score = scores[static_cast<size_t>(idx) * stride];
      e.id = ids != nullptr ? ids[idx] : static_cast<int64_t>(idx);
      e.index = idx;
      e.pad = 0;
      buf[i] = e;
    } else {
      buf[i] = sentinel();
    }
  }
  bitonic_sort(buf, P);
  for (int j = threadIdx.x; j < k; j += blockDim.x) dst[j] = j < P ? buf[j] : sentinel();
}

// Stage 2 / merge: segment s owns entries in[s*per_seg .. (s+1)*per_seg),
// entries at or past n_total (a partial last segment) read as sentinels.
__global__ void __launch_bounds__(kSortThreads)
    topk_entries_kernel(const TopkEntry* __restrict__ in, int per_seg, int k,
                        TopkEntry* __restrict__ out, long long n_total) {
  pdl_wait();
  extern __shared__ TopkEntry buf[];
  const long long seg0 = static_cast<long long>(blockIdx.x) * per_seg;
  const TopkEntry* src = in + seg0;
  const int P = pow2_at_least(per_seg);
  for (int i = threadIdx.x; i < P; i += blockDim.x)
    buf[i] = (i < per_seg && seg0 + i < n_total) ? src[i] : sentinel();
  bitonic_sort(buf, P);
  TopkEntry* dst = out + static_cast<size_t>(blockIdx.x) * k;
  for (int j = threadIdx.x; j < k; j += blockDim.x) dst[j] = j < P ? buf[j] : sentinel();
}

// Output side of the service (service.cpp:242-277): calibrate() of the
// relevance (calibration.cpp:65-88: clamp(value) of the block holding the
// score, linear ramp across gaps), then the final score = calibrated
// relevance, or sum_j w_j * calibrated[task_j] in the caller's (std::map)
// order. Same double operations in the same order as the reference.
__global__ void final_score_kernel(const double* __restrict__ scores, int stride, int n,
                                   const double* __restrict__ blk, int n_blocks,
                                   const int32_t* __restrict__ blend_task,
                                   const double* __restrict__ blend_w, int n_blend,
                                   double* __restrict__ out) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double raw = scores[static_cast<size_t>(i) * stride];
  double cal = raw;
  if (n_blocks > 0) {
    auto lo = [&](int b) { return blk[3 * b]; };
    auto hi = [&](int b) { return blk[3 * b + 1]; };
    auto val = [&](int b) { return blk[3 * b + 2]; };
    auto clamp01 = [](double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); };
    if (raw <= hi(0)) {
      cal = clamp01(val(0));
    } else {
      cal = clamp01(val(n_blocks - 1));
      for (int b = 0; b + 1 < n_blocks; ++b) {
        if (raw < lo(b + 1)) {
          const double t = __ddiv_rn(__dsub_rn(raw, hi(b)), __dsub_rn(lo(b + 1), hi(b)));
          cal = clamp01(__dadd_rn(val(b), __dmul_rn(t, __dsub_rn(val(b + 1), val(b)))));
          break;
        }
        if (raw <= hi(b + 1)) {
          cal = clamp01(val(b + 1));
          break;
        }
      }
    }
  }
  double f = cal;
  if (n_blend > 0) {
    f = 0.0;
    for (int j = 0; j < n_blend; ++j) {
      const int tk = blend_task[j];
      const double v = tk == 0 ? cal : scores[static_cast<size_t>(i) * stride + tk];
      f = __dadd_rn(f, __dmul_rn(blend_w[j], v));
    }
  }
  out[i] = f;
  pdl_trigger();
}

}  // namespace

cudaError_t final_scores(const double* scores, int stride, int n, const double* blocks,
                         int n_blocks, const int32_t* blend_task, const double* blend_w,
                         int n_blend, double* out, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  return launch_k(final_score_kernel, dim3((n + 255) / 256), dim3(256), 0, stream, scores, stride,
                  n, blocks, n_blocks, blend_task, blend_w, n_blend, out);
}

cudaError_t score_head(const float* x, const int32_t* last_rows, int n_items, int d,
                       const float* ln_gain, const float* w_cols, const float* bias, int n_cols,
                       const int32_t* task_col, const int32_t* task_arity, int n_tasks,
                       int yes_col, int no_col, double* scores, float* hidden_out,
                       cudaStream_t stream) {
  if (n_items <= 0) return cudaSuccess;
  if (d % 4 != 0) return cudaErrorInvalidValue;
  const int nv = (d / 4 + 31) / 32;
#define SRK_HEAD(NVV)                                                                        \
  return launch_head<NVV>(x, last_rows, n_items, d, ln_gain, w_cols, bias, n_cols, task_col, \
                          task_arity, n_tasks, yes_col, no_col, scores, hidden_out, stream)
  if (nv <= 1) SRK_HEAD(1);
  if (nv <= 2) SRK_HEAD(2);
  if (nv <= 4) SRK_HEAD(4);
  if (nv <= 8) SRK_HEAD(8);
  if (nv <= 16) SRK_HEAD(16);
  if (nv <= 32) SRK_HEAD(32);
#undef SRK_HEAD
  return cudaErrorInvalidValue;
}

cudaError_t topk(const double* scores, int stride, const int64_t* ids, const int32_t* seg_off,
                 int n_segments, int max_seg_len, int k, TopkEntry* scratch, int scratch_cap,
                 TopkEntry* out, cudaStream_t stream) {
  if (n_segments <= 0 || k <= 0) return cudaSuccess;
  if (k > kSortCap) return cudaErrorInvalidValue;
  const int chunks = (max_seg_len + kSortCap - 1) / kSortCap;
  const size_t smem = sizeof(TopkEntry) * kSortCap;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(topk_scores_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    cudaFuncSetAttribute(topk_entries_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    attr = true;
  }
  if (chunks <= 1) {
    return launch_k(topk_scores_kernel, dim3(n_segments), dim3(kSortThreads), smem, stream, scores,
                    stride, ids, seg_off, n_segments, k, out, 1);
  }
  if (static_cast<long>(chunks) * k > kSortCap) return cudaErrorInvalidValue;
  if (static_cast<long>(n_segments) * chunks * k > scratch_cap) return cudaErrorInvalidValue;
  cudaError_t e = launch_k(topk_scores_kernel, dim3(n_segments * chunks), dim3(kSortThreads), smem,
                           stream, scores, stride, ids, seg_off, n_segments, k, scratch, chunks);
  if (e != cudaSuccess) return e;
  return launch_k(topk_entries_kernel, dim3(n_segments), dim3(kSortThreads), smem, stream,
                  static_cast<const TopkEntry*>(scratch), chunks * k, k, out,
                  static_cast<long long>(n_segments) * chunks * k);
}

cudaError_t topk_merge(const TopkEntry* in, int n, int k, TopkEntry* out, cudaStream_t stream) {
  if (n <= 0 || k <= 0) return cudaSuccess;
  if (n > kSortCap) return cudaErrorInvalidValue;
  const size_t smem = sizeof(TopkEntry) * kSortCap;
  cudaFuncSetAttribute(topk_entries_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  return launch_k(topk_entries_kernel, dim3(1), dim3(kSortThreads), smem, stream, in, n, k, out,
                  static_cast<long long>(n));
}

// Group size of the reduction levels: the bitonic sort cost grows as
// G log^2 G per CTA and a level runs ceil(m / G) CTAs side by side, so small
// groups (8k, at least 256) finish far sooner than 4096-entry ones (a 200k-doc
// retrieval query: 120 us -> ~25 us of selection). Each level keeps k of G.
static int select_group(int k) {
  int g = 256;
  while (g < 8 * k && g < kSortCap) g <<= 1;
  return g;
}

size_t topk_select_scratch(long long n, int k) {
  // level sizes shrink by >= 2x (groups of G entries -> k each, k <= G / 2)
  const int G = select_group(k);
  size_t total = 0;
  long long m = n;
  while (m > G) {
    const long long groups = (m + G - 1) / G;
    m = groups * k;
    total += static_cast<size_t>(m);
  }
  return total + 1;
}

cudaError_t topk_select(const TopkEntry* in, long long n, int k, TopkEntry* scratch,
                        TopkEntry* out, cudaStream_t stream) {
  if (n <= 0 || k <= 0) return cudaSuccess;
  if (k > kSortCap / 2) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(topk_entries_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(TopkEntry) * kSortCap));
    attr = true;
  }
  const int G = select_group(k);
  const TopkEntry* cur = in;
  long long m = n;
  TopkEntry* dst = scratch;
  while (m > G) {
    const long long groups = (m + G - 1) / G;
    cudaError_t e = launch_k(topk_entries_kernel, dim3(static_cast<unsigned>(groups)),
                             dim3(kSortThreads), sizeof(TopkEntry) * G, stream, cur, G, k, dst, m);
    if (e != cudaSuccess) return e;
    cur = dst;
    m = groups * k;
    dst += m;
  }
  const int mm = static_cast<int>(m);
  int P = 1;
  while (P < mm) P <<= 1;
  return launch_k(topk_entries_kernel, dim3(1), dim3(kSortThreads), sizeof(TopkEntry) * P, stream,
                  cur, mm, k, out, m);
}

}  // namespace srk
