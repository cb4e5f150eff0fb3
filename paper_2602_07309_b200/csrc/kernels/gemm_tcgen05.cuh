// Persistent, warp-specialised bf16 GEMM on 5th-generation tensor cores.
//
//   C[M x N] = A[M x K] . B[N x K]^T     (A = activations, B = W^T, both K-major)
//
// Replaces the reference's fp32 row-loop matmul (kernels.cpp:16-29, 101-125)
// for the four per-layer projections (model.cpp:189-213). Epilogues fuse the
// element-wise work that follows each projection in the reference:
//   EPI_BF16      Q|K|V projection -> bf16 (model.cpp:189-196)
//   EPI_GELU_BF16 W_in + exact-erf GELU -> bf16 (model.cpp:206-209, kernels.cpp:47-49)
//   EPI_RESID_F32 x += acc, fp32 residual stream (model.cpp:199-202, 210-213)
//   EPI_F32       plain fp32 store (tests)
//
// Roles (192 threads, one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: A/B k-blocks into a STAGES-deep smem ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> fused op -> HBM
// The accumulator is double-buffered in TMEM (2 x BN fp32 columns) so the
// epilogue of tile i overlaps the main loop of tile i+1.
#pragma once

#include "ptx.cuh"

namespace srk {

enum GemmEpilogue : int { EPI_BF16 = 0, EPI_GELU_BF16 = 1, EPI_RESID_F32 = 2, EPI_F32 = 3 };

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;  // 64 bf16 = one 128-byte swizzle row
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN >= 256) ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int TMEM_COLS = 2 * BN;  // power of two for BN in {64,128,256}
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 256 + 1024;
  static constexpr int THREADS = 192;
};

template <int BN, int EPI>
__global__ void __launch_bounds__(192, 1)
    gemm_bf16_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA,
                             const __grid_constant__ CUtensorMap tmB, int M, int N, int K,
                             void* __restrict__ out, int ldo) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_tiles = (M + C::BM - 1) / C::BM;
  const int n_tiles = N / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int nk = (K + C::BK - 1) / C::BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // Weights (B) are re-read by every M tile: keep them in L2.
      const uint64_t pol_b = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int m0 = (tile / n_tiles) * C::BM;
        const int n0 = (tile % n_tiles) * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_2d(&tmA, &full[stage], sA + stage * C::A_BYTES, kb * C::BK, m0);
          tma_load_2d_hint(&tmB, &full[stage], sB + stage * C::B_BYTES, kb * C::BK, n0, pol_b);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(C::BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k) {
            // Advancing K by 16 elements = 32 bytes inside the 128 B swizzle row.
            umma_bf16(d_tmem, sw128_kmajor_desc(a_addr + k * 32),
                      sw128_kmajor_desc(b_addr + k * 32), idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // Epilogue: warp w may only touch TMEM lanes [32*(w%4), 32*(w%4)+32).
    const int quad = warp & 3;
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int m0 = (tile / n_tiles) * C::BM;
      const int n0 = (tile % n_tiles) * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int row = m0 + quad * 32 + lane;
      const bool live = row < M;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN + c,
                           r);
        tmem_ld_wait();
        if (!live) continue;
        const size_t off = static_cast<size_t>(row) * ldo + n0 + c;
        if constexpr (EPI == EPI_BF16 || EPI == EPI_GELU_BF16) {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + off);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              f[j] = __uint_as_float(r[v * 8 + j]);
              if constexpr (EPI == EPI_GELU_BF16) f[j] = gelu_erf(f[j]);
            }
            dst[v] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                                pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
          }
        } else if constexpr (EPI == EPI_RESID_F32) {
          float4* x = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + off);
          float4 cur[8];
#pragma unroll
          for (int v = 0; v < 8; ++v) cur[v] = x[v];
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            cur[v].x += __uint_as_float(r[v * 4 + 0]);
            cur[v].y += __uint_as_float(r[v * 4 + 1]);
            cur[v].z += __uint_as_float(r[v * 4 + 2]);
            cur[v].w += __uint_as_float(r[v * 4 + 3]);
            x[v] = cur[v];
          }
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + off);
#pragma unroll
          for (int v = 0; v < 8; ++v)
            dst[v] = make_float4(__uint_as_float(r[v * 4 + 0]), __uint_as_float(r[v * 4 + 1]),
                                 __uint_as_float(r[v * 4 + 2]), __uint_as_float(r[v * 4 + 3]));
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem_base, C::TMEM_COLS);
}

}  // namespace srk
