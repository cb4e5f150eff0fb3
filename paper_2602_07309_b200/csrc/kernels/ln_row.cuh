// One LayerNorm row held by a warp (reference kernels.cpp:31-45: two-pass
// mean / population variance, eps 1e-5, gain only), shared by the row
// kernels (rowops.cu) and the residual GEMM's LN-after epilogue
// (gemm_tcgen05.cuh, EPI_RESID_F32_LN) so both produce identical bits.
#pragma once

#include <cuda_bf16.h>

namespace srk {

constexpr float kLnEps = 1e-5f;

// Row held as float4 chunks: lane owns chunks lane, lane+32, ...
template <int NV>
__device__ __forceinline__ void ln_row_store(const float4 (&v)[NV], int d4, const float* gain,
                                             __nv_bfloat16* out_row, int lane) {
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < d4) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffff, s, o);
  const float d = static_cast<float>(d4 * 4);
  const float mean = s / d;
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
  const float inv = 1.0f / sqrtf(q / d + kLnEps);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + i * 32;
    if (c < d4) {
      const float4 gg = reinterpret_cast<const float4*>(gain)[c];
      uint2 packed;
      __nv_bfloat162 lo = __floats2bfloat162_rn((v[i].x - mean) * inv * gg.x,
                                                (v[i].y - mean) * inv * gg.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn((v[i].z - mean) * inv * gg.z,
                                                (v[i].w - mean) * inv * gg.w);
      packed.x = *reinterpret_cast<uint32_t*>(&lo);
      packed.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(out_row)[c] = packed;
    }
  }
}

}  // namespace srk
