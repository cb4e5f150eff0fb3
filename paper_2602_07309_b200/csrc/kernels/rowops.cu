// Row kernels: embedding gather (+ fused layer-0 LN1), gain-only LayerNorm,
// and the one-time weight conversion fp32 [K x N] -> bf16 [N x K].
//
// LayerNorm semantics follow kernels.cpp:31-45 (layer_norm_row): two-pass
// mean then population variance, eps 1e-5, (x - mean) * rsqrt(var + eps) * gain,
// no bias. One warp per row; the row lives in registers between passes, so
// HBM traffic is one fp32 read + one bf16 write per element.
#include <cuda_bf16.h>

#include <algorithm>

#include "launch.h"
#include "ln_row.cuh"
#include "ptx.cuh"

namespace srk {

namespace {

template <int NV>
__global__ void __launch_bounds__(256)
    embed_ln_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ pos,
                    const float* __restrict__ tok_emb, const float* __restrict__ soft_rows,
                    const float* __restrict__ pos_emb, const float* __restrict__ gain,
                    float* __restrict__ x, __nv_bfloat16* __restrict__ xn, int M, int d) {
  pdl_wait();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const int d4 = d >> 2;
  const int s = src[row];
  const float4* e = reinterpret_cast<const float4*>(
      s >= 0 ? tok_emb + static_cast<size_t>(s) * d
             : soft_rows + static_cast<size_t>(-s - 1) * d);
  const float4* p = reinterpret_cast<const float4*>(pos_emb + static_cast<size_t>(pos[row]) * d);
  float4* xr = reinterpret_cast<float4*>(x + static_cast<size_t>(row) * d);
  float4 v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < d4) {
      const float4 a = e[c], b = p[c];
      // model.cpp:258-271 / 282-290: rows = embedding + pos_emb, fp32
      v[i] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
      xr[c] = v[i];
    }
  }
  ln_row_store<NV>(v, d4, gain, xn + static_cast<size_t>(row) * d, lane);
  pdl_trigger();
}

// Folded-LN variant (gemm_tcgen05.cuh GemmLnArgs): the layer-0 LN1 is
// finished inside the QKV GEMM, so this writes x, xb = bf16(x) and the row's
// (mean, M2) (two-pass, as kernels.cpp:31-45) as the single statistics part.
template <int NV>
__global__ void __launch_bounds__(256)
    embed_stats_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ pos,
                       const float* __restrict__ tok_emb, const float* __restrict__ soft_rows,
                       const float* __restrict__ pos_emb, float* __restrict__ x,
                       __nv_bfloat16* __restrict__ xb, float2* __restrict__ stats, int M, int d) {
  pdl_wait();
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const int d4 = d >> 2;
  const int s = src[row];
  const float4* e = reinterpret_cast<const float4*>(
      s >= 0 ? tok_emb + static_cast<size_t>(s) * d
             : soft_rows + static_cast<size_t>(-s - 1) * d);
  const float4* p = reinterpret_cast<const float4*>(pos_emb + static_cast<size_t>(pos[row]) * d);
  float4* xr = reinterpret_cast<float4*>(x + static_cast<size_t>(row) * d);
  uint2* br = reinterpret_cast<uint2*>(xb + static_cast<size_t>(row) * d);
  float4 v[NV];
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < d4) {
      const float4 a = e[c], b = p[c];
      v[i] = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
      xr[c] = v[i];
      __nv_bfloat162 lo = __floats2bfloat162_rn(v[i].x, v[i].y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(v[i].z, v[i].w);
      br[c] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
      sum += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffff, sum, o);
  const float mean = sum / static_cast<float>(d);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < d4) {
      const float a = v[i].x - mean, b = v[i].y - mean, g = v[i].z - mean, h = v[i].w - mean;
      q += (a * a + b * b) + (g * g + h * h);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffff, q, o);
  if (lane == 0) stats[row] = make_float2(mean, q);
  pdl_trigger();
}

template <int NV>
cudaError_t launch_embed_stats(const int32_t* src, const int32_t* pos, const float* tok_emb,
                               const float* soft_rows, const float* pos_emb, float* x,
                               __nv_bfloat16* xb, float* stats, int M, int d,
                               cudaStream_t stream) {
  return launch_k(embed_stats_kernel<NV>, dim3((M + 7) / 8), dim3(256), 0, stream, src, pos,
                  tok_emb, soft_rows, pos_emb, x, xb, reinterpret_cast<float2*>(stats), M, d);
}

// One warp per weight row: out[n] = sum_k float(w[n][k]) (double accumulation).
__global__ void bf16_row_sums_kernel(const __nv_bfloat16* __restrict__ w, int N, int K,
                                     float* __restrict__ out) {
  const int n = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  double s = 0.0;
  for (int k = lane; k < K; k += 32) s += static_cast<double>(__bfloat162float(w[static_cast<size_t>(n) * K + k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  if (lane == 0) out[n] = static_cast<float>(s);
}

// Rows (one warp each) per LayerNorm CTA (C2, 3 interleaved rounds: 4 rows
// 1.07 ms, 8 rows 1.05-1.08 ms, 16 rows 1.15-1.16 ms per query).
#ifndef SRK_LN_ROWS
#define SRK_LN_ROWS 8
#endif

template <int NV>
__global__ void __launch_bounds__(SRK_LN_ROWS * 32)
    layer_norm_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                      __nv_bfloat16* __restrict__ out, int M, int d, int rev) {
  pdl_wait();
  const int blk = rev ? gridDim.x - 1 - blockIdx.x : blockIdx.x;
  const int row = blk * SRK_LN_ROWS + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= M) return;
  const int d4 = d >> 2;
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<size_t>(row) * d);
  float4 v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < d4) v[i] = xr[c];
  }
  ln_row_store<NV>(v, d4, gain, out + static_cast<size_t>(row) * d, lane);
  pdl_trigger();
}

// Polls the residual GEMM's per-block completion counts (epi 7) and
// normalises each 128-row block as soon as its add-reductions are complete,
// reading x while it is still in L2. Blocks are visited in the GEMM's tile
// order (increasing), one CTA per SM, 8 warps x 16 rows per block.
template <int NV>
__global__ void __launch_bounds__(256)
    layer_norm_after_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                            __nv_bfloat16* __restrict__ out, int M, int d,
                            unsigned int* __restrict__ cnt, unsigned int contrib) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = (M + 127) / 128;
  const int d4 = d >> 2;
  for (int b = blockIdx.x; b < nblk; b += gridDim.x) {
    if (threadIdx.x == 0) {
      unsigned int v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt + b) : "memory");
        if (v >= contrib) break;
        __nanosleep(256);
      }
    }
    __syncthreads();
    const int r0 = b * 128 + warp * 16;
#pragma unroll 1
    for (int rr = 0; rr < 16; rr += 2) {
      float4 v0[NV], v1[NV];
      const int ra = r0 + rr, rb = ra + 1;
      const float4* xa = reinterpret_cast<const float4*>(x + static_cast<size_t>(ra) * d);
      const float4* xb = reinterpret_cast<const float4*>(x + static_cast<size_t>(rb) * d);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int c = lane + 32 * i;
        if (ra < M && c < d4) v0[i] = ld_cg_f4(xa + c);
        if (rb < M && c < d4) v1[i] = ld_cg_f4(xb + c);
      }
      if (ra < M) ln_row_store<NV>(v0, d4, gain, out + static_cast<size_t>(ra) * d, lane);
      if (rb < M) ln_row_store<NV>(v1, d4, gain, out + static_cast<size_t>(rb) * d, lane);
    }
    __syncthreads();
    if (threadIdx.x == 0) cnt[b] = 0u;  // ready for the next residual GEMM (stream-ordered)
  }
}

template <int NV>
cudaError_t launch_ln_after(const float* x, const float* gain, __nv_bfloat16* out, int M, int d,
                            unsigned int* cnt, int contrib, cudaStream_t stream) {
  // one CTA per block (several per SM next to the GEMM's CTA: more rows in
  // flight per SM than one persistent CTA could keep)
  const int nblk = (M + 127) / 128;
  const int grid = nblk;
  layer_norm_after_kernel<NV><<<grid, 256, 0, stream>>>(x, gain, out, M, d, cnt,
                                                        static_cast<unsigned int>(contrib));
  return cudaGetLastError();
}

template <int NV>
cudaError_t launch_embed(const int32_t* src, const int32_t* pos, const float* tok_emb,
                         const float* soft_rows, const float* pos_emb, const float* gain, float* x,
                         __nv_bfloat16* xn, int M, int d, cudaStream_t stream) {
  return launch_k(embed_ln_kernel<NV>, dim3((M + 7) / 8), dim3(256), 0, stream, src, pos, tok_emb,
                  soft_rows, pos_emb, gain, x, xn, M, d);
}

template <int NV>
cudaError_t launch_ln(const float* x, const float* gain, __nv_bfloat16* out, int M, int d,
                      cudaStream_t stream, int rev) {
  return launch_k(layer_norm_kernel<NV>, dim3((M + SRK_LN_ROWS - 1) / SRK_LN_ROWS),
                  dim3(SRK_LN_ROWS * 32), 0, stream, x, gain, out, M,
                  d, rev);
}

__global__ void transpose_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                      int K, int N, const float* __restrict__ scale_k) {
  __shared__ float tile[32][33];
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int k = k0 + i, n = n0 + threadIdx.x;
    tile[i][threadIdx.x] = (k < K && n < N) ? src[static_cast<size_t>(k) * N + n] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int n = n0 + i, k = k0 + threadIdx.x;
    if (n < N && k < K)
      dst[static_cast<size_t>(n) * K + k] =
          __float2bfloat16_rn(scale_k ? tile[threadIdx.x][i] * scale_k[k] : tile[threadIdx.x][i]);
  }
}

}  // namespace

#define SRK_DISPATCH_NV(d, FN, ...)              \
  do {                                           \
    const int nv = ((d) / 4 + 31) / 32;          \
    if (nv <= 1) return FN<1>(__VA_ARGS__);      \
    if (nv <= 2) return FN<2>(__VA_ARGS__);      \
    if (nv <= 4) return FN<4>(__VA_ARGS__);      \
    if (nv <= 8) return FN<8>(__VA_ARGS__);      \
    if (nv <= 16) return FN<16>(__VA_ARGS__);    \
    if (nv <= 32) return FN<32>(__VA_ARGS__);    \
    return cudaErrorInvalidValue;                \
  } while (0)

cudaError_t embed_ln(const int32_t* src, const int32_t* pos, const float* tok_emb,
                     const float* soft_rows, const float* pos_emb, const float* gain, float* x,
                     __nv_bfloat16* xn, int M, int d, cudaStream_t stream) {
  if (M <= 0) return cudaSuccess;
  if (d % 4 != 0) return cudaErrorInvalidValue;
  SRK_DISPATCH_NV(d, launch_embed, src, pos, tok_emb, soft_rows, pos_emb, gain, x, xn, M, d,
                  stream);
}

cudaError_t layer_norm_bf16(const float* x, const float* gain, __nv_bfloat16* out, int M, int d,
                            cudaStream_t stream, bool rev) {
  if (M <= 0) return cudaSuccess;
  if (d % 4 != 0) return cudaErrorInvalidValue;
  SRK_DISPATCH_NV(d, launch_ln, x, gain, out, M, d, stream, rev ? 1 : 0);
}

cudaError_t layer_norm_after(const float* x, const float* gain, __nv_bfloat16* out, int M, int d,
                             unsigned int* cnt, int contrib, cudaStream_t stream) {
  if (M <= 0) return cudaSuccess;
  if (d % 4 != 0 || cnt == nullptr || contrib <= 0) return cudaErrorInvalidValue;
  SRK_DISPATCH_NV(d, launch_ln_after, x, gain, out, M, d, cnt, contrib, stream);
}

cudaError_t transpose_to_bf16(const float* src, __nv_bfloat16* dst, int K, int N,
                              cudaStream_t stream, const float* scale_k) {
  dim3 grid((N + 31) / 32, (K + 31) / 32), block(32, 8);
  transpose_bf16_kernel<<<grid, block, 0, stream>>>(src, dst, K, N, scale_k);
  return cudaGetLastError();
}

cudaError_t bf16_row_sums(const __nv_bfloat16* w, int N, int K, float* out, cudaStream_t stream) {
  if (N <= 0) return cudaSuccess;
  bf16_row_sums_kernel<<<(N + 7) / 8, 256, 0, stream>>>(w, N, K, out);
  return cudaGetLastError();
}

// Compact per-item embeddings -> soft-token rows (mixed mode).
// Zero-pad form (service.cpp:208-217): row i = emb[i][0 .. min(d_emb, d)), 0 after.
__global__ void emb_pad_rows_kernel(const float* __restrict__ emb, int n, int d_emb, int d,
                                    float* __restrict__ out) {
  const long long total = static_cast<long long>(n) * d;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(t / d), j = static_cast<int>(t % d);
    out[t] = j < d_emb ? emb[static_cast<long long>(i) * d_emb + j] : 0.f;
  }
}

// Projection operand: bf16 rows [n x kp], columns >= d_emb zero.
__global__ void emb_to_bf16_kernel(const float* __restrict__ emb, int n, int d_emb, int kp,
                                   __nv_bfloat16* __restrict__ out) {
  const long long total = static_cast<long long>(n) * kp;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(t / kp), j = static_cast<int>(t % kp);
    out[t] = __float2bfloat16_rn(j < d_emb ? emb[static_cast<long long>(i) * d_emb + j] : 0.f);
  }
}

cudaError_t emb_pad_rows(const float* emb, int n, int d_emb, int d, float* out,
                         cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const long long total = static_cast<long long>(n) * d;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  emb_pad_rows_kernel<<<blocks, 256, 0, stream>>>(emb, n, d_emb, d, out);
  return cudaGetLastError();
}

cudaError_t emb_to_bf16(const float* emb, int n, int d_emb, int kp, __nv_bfloat16* out,
                        cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const long long total = static_cast<long long>(n) * kp;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148 * 16));
  emb_to_bf16_kernel<<<blocks, 256, 0, stream>>>(emb, n, d_emb, kp, out);
  return cudaGetLastError();
}

cudaError_t embed_stats(const int32_t* src, const int32_t* pos, const float* tok_emb,
                        const float* soft_rows, const float* pos_emb, float* x,
                        __nv_bfloat16* xb, float* stats, int M, int d, cudaStream_t stream) {
  if (M <= 0) return cudaSuccess;
  if (d % 4 != 0) return cudaErrorInvalidValue;
  SRK_DISPATCH_NV(d, launch_embed_stats, src, pos, tok_emb, soft_rows, pos_emb, x, xb, stats, M,
                  d, stream);
}

}  // namespace srk
