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
// Roles (320 threads, one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: A/B k-blocks into a STAGES-deep smem ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..9  epilogue, two warps per TMEM lane quadrant (column halves):
//               tcgen05.ld -> registers -> fused op -> 32-row x 128 B chunk in
//               a swizzled smem staging buffer -> TMA bulk store, or for the
//               residual a TMA bulk add-reduction (the L2 performs x += acc in
//               fp32, so the SM never reads x and every access is a full line).
// The accumulator is double-buffered in TMEM (2 x BN fp32 columns) so the
// epilogue of tile i overlaps the main loop of tile i+1.
#pragma once

#include "launch.h"
#include "ptx.cuh"

namespace srk {

// GemmEpilogue (EPI_*) is declared in launch.h.

// Optional per-CTA timeline of the pair kernel (%globaltimer ns, 64 slots per
// CTA): 0 entry, 1 setup done, 2+i MMA of local tile i issued, 24+i epilogue
// of tile i done, 63 exit. Kernel tuning only (sr_debug_gemm_trace).
__device__ unsigned long long* g_gemm_trace = nullptr;
__device__ __forceinline__ void gemm_trace(int slot) {
  if (g_gemm_trace != nullptr && blockIdx.x < 256) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gemm_trace[blockIdx.x * 64 + slot] = t;
  }
}

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;  // 64 bf16 = one 128-byte swizzle row
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN >= 256) ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int TMEM_COLS = 2 * BN;  // power of two for BN in {64,128,256}
  static constexpr int EPI_WARPS = 8;       // two per TMEM lane quadrant (column halves)
  static constexpr int STG_BYTES = 32 * 128;  // per epilogue warp: 32 rows x 128 B
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_WARPS * STG_BYTES + 256 + 1024;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
};

// Output tensor map box for an epilogue: 32 rows x 128 B (32 fp32 or 64 bf16).
template <int EPI>
struct EpiOut {
  static constexpr bool F32 =
      (EPI == EPI_RESID_F32 || EPI == EPI_F32 || EPI == EPI_RESID_LN || EPI == EPI_RESID_F32_LN);
  static constexpr int CW = F32 ? 32 : 64;  // columns per staged chunk
};

template <int BN, int EPI>
__global__ void __launch_bounds__(320, 1)
    gemm_bf16_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA,
                             const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmC, int M, int N, int K) {
  using C = GemmCfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sStg = sB + C::STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + C::EPI_WARPS * C::STG_BYTES);
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
    tma_prefetch_desc(&tmC);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 32 * C::EPI_WARPS);
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
  pdl_wait();  // inputs of the previous kernel (and its reads of our outputs) are done

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
    // Epilogue: warp w may only touch TMEM lanes [32*(w%4), 32*(w%4)+32);
    // the two warps of a quadrant split the tile's columns.
    constexpr int CW = EpiOut<EPI>::CW;
    constexpr int SPAN = (BN / 2 > CW) ? BN / 2 : CW;  // columns per warp
    const int quad = warp & 3;
    const int col0 = ((warp - 2) >> 2) * SPAN;
    uint8_t* stg = sStg + (warp - 2) * C::STG_BYTES;
    const uint64_t pol_keep = policy_evict_last();
    int local = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int m0 = (tile / n_tiles) * C::BM;
      const int n0 = (tile % n_tiles) * BN;
      const int r0 = m0 + quad * 32;  // first row of this warp's 32-row slab
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (col0 < BN && r0 < M) {
#pragma unroll 1
        for (int c = col0; c < col0 + SPAN; c += CW) {
          // the staging buffer is free once the previous bulk op read it
          if (lane == 0) bulk_wait_read0();
          __syncwarp();
          uint8_t* row_base = stg + lane * 128;
          if constexpr (EpiOut<EPI>::F32) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN + c,
                               r);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 8; ++k)
              *reinterpret_cast<uint4*>(row_base + ((k ^ (lane & 7)) * 16)) =
                  make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
          } else {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              uint32_t r[32];
              tmem_ld_32x32b_x32(
                  tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN + c + hh * 32, r);
              tmem_ld_wait();
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                float f[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  f[j] = __uint_as_float(r[8 * k + j]);
                  if constexpr (EPI == EPI_GELU_BF16) f[j] = gelu_erf(f[j]);
                }
                const int chunk = hh * 4 + k;
                *reinterpret_cast<uint4*>(row_base + ((chunk ^ (lane & 7)) * 16)) =
                    make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                               pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
              }
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if constexpr (EPI == EPI_RESID_F32)  // x is re-read next by the LayerNorm
              tma_reduce_add_2d_hint(&tmC, stg, n0 + c, r0, pol_keep);
            else
              tma_store_2d(&tmC, stg, n0 + c, r0);
            bulk_commit();
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
    if (lane == 0) bulk_wait0();
  }

  pdl_trigger();  // this CTA's work is issued: the next kernel may start launching
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem_base, C::TMEM_COLS);
}

// ----------------------------------------------------------------------------
// LayerNorm folded into the GEMMs (pair kernel only).
//
// The reference normalises the residual stream before each projection
// (model.cpp:187-188, 204-205: h = LN(x) * gain, then h . W). Here LN never
// materialises:
//   * the residual GEMMs (O and W_out, EPI_RESID_LN) load the fp32 x tile,
//     add the accumulator, store x, store a bf16 copy xb, and write per-row
//     partial statistics (mean, M2) over each 128-column slice;
//   * the next projection (QKV / W_in, EPI_LN_BF16 / EPI_LN_GELU_BF16) takes
//     xb as its A operand against gain-folded weights W' = diag(gain) W and
//     finishes the normalisation in the epilogue:
//         LN(x) . W' = rstd * (xb . W' - mean * colsum(W'))
//     with mean/rstd combined from the partials (Chan et al.), i.e. the
//     reference's two-pass population variance and eps 1e-5 (kernels.cpp:31-45).
struct alignas(64) GemmLnArgs {
  CUtensorMap tm_xb;        // EPI_RESID_LN: bf16 copy of x, 32 x 64 boxes, 128 B swizzle
  float2* stats_out;        // EPI_RESID_LN: [N / 128][ld] (mean, M2) over 128 columns
  const float2* stats_in;   // EPI_LN_*: [n_parts][ld], each part over K / n_parts columns
  const float* colsum;      // EPI_LN_*: [N] column sums of the folded bf16 weights
  unsigned int* ln_cnt;     // EPI_RESID_F32_LN: per 128-row block add-reductions done
  float* resid_out;         // EPI_RESID_F32 (SRK_RESID_RED): x [M x ld] for red.global.add
  int resid_ld;
  int n_parts;
  int ld;
};

// ----------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs on one TPC computes a
// 256 x 256 tile; CTA r loads rows [128 r, +128) of A and of B (= 128 of the
// 256 output columns) per k-block, the leader issues
// tcgen05.mma.cta_group::2 (M = 256) which reads both CTAs' smem and writes
// each CTA's 128 accumulator rows into its own TMEM. Per SM this halves the
// B operand traffic through shared memory relative to the 1-CTA 128 x 256
// tile (the 1-CTA kernel is smem-bandwidth bound at ~64% tensor-pipe).
//
// NP = 2 pairs per cluster (cluster of 4): the two pairs compute adjacent
// 256-column tiles of the same 256 rows, so each A k-block is fetched once
// and multicast to both pairs (pair kb % 2 issues it): a quarter less L2 ->
// SM operand traffic, at the cost of the SMs a 4-CTA cluster grid cannot use
// (132 of 148 on B200). Opt-in (SRK_GEMM_NP=2): on the C2 shapes the per-tile
// time did not change, so NP = 1 on all 148 SMs is faster.
#ifndef SRK_PAIR_STAGES
#define SRK_PAIR_STAGES 6
#endif
#ifndef SRK_PAIR_STG_BUFS
#define SRK_PAIR_STG_BUFS 1
#endif
// Tail split of the pair GEMM's last wave (see the kernel). Opt-in: the O /
// W_out classes get 4-5% faster in the per-class replay, but the pipelined
// C2 step measured slower (8.94-9.09 vs 8.84-8.88 ms, 4 interleaved rounds).
// Residual epilogue by vector reductions from registers (REDG.ADD.F32x4)
// instead of smem staging + TMA add-reduce. Motivation (tools/gemm_trace.py,
// C2): the staged reduction's shared-memory traffic stretches the O GEMM's
// main loop from 6.1 (bf16-epilogue GEMMs of the same K) to 8.5 us per tile.
// Measured: the register path needs 11.7 us per tile of epilogue (=1: 32x32b
// loads, 32 rows x 16 B per warp reduction) or 8.3 us (=2: 16x256b loads, 8
// rows x one full 32 B sector per warp reduction) against 3.65 us staged, so
// the GEMM turns epilogue-bound: O / W_out 1.84 / 2.02 (=1), 1.49 / 1.78 (=2)
// vs 1.30 / 1.68 ms per query. Off.
#ifndef SRK_RESID_RED
#define SRK_RESID_RED 0
#endif
#ifndef SRK_TAIL_SPLIT
#define SRK_TAIL_SPLIT 0
#endif
#ifndef SRK_RESID_LN_STAGES
#define SRK_RESID_LN_STAGES 5
#endif
// EPI_RESID_F32 (O / W_out add-reduction epilogue): staging buffers per
// epilogue warp and ring depth (2 buffers let chunk c's reduction overlap the
// TMEM drain of chunk c + 1, paid for with one ring stage).
#ifndef SRK_RESID_STG_BUFS
#define SRK_RESID_STG_BUFS SRK_PAIR_STG_BUFS
#endif
#ifndef SRK_RESID_STAGES
#define SRK_RESID_STAGES SRK_PAIR_STAGES
#endif
template <int EPI>
struct GemmPairCfg {
  static constexpr int BM = 128;  // rows per CTA (pair: 256)
  static constexpr int BN = 256;  // output columns per pair tile
  static constexpr int BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;        // 16 KB
  static constexpr int B_BYTES = (BN / 2) * BK * 2;  // 16 KB (this CTA's half of B)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // The residual+LN epilogue stages x in and out (1 fp32 chunk + 1 bf16
  // chunk per warp), paid for with one ring stage. (A register -> global
  // variant with 16x256b TMEM loads was measured slower: 8 rows x 32 B per
  // store instruction made the epilogue LSU-bound, 2-3x the staged time.)
  static constexpr bool RESID_LN = EPI == EPI_RESID_LN;
  static constexpr bool RESID_F32 = EPI == EPI_RESID_F32 || EPI == EPI_RESID_F32_LN;
  static constexpr int STAGES =
      RESID_LN ? SRK_RESID_LN_STAGES : (RESID_F32 ? SRK_RESID_STAGES : SRK_PAIR_STAGES);
  static constexpr int TMEM_COLS = 2 * BN;  // double-buffered 128 x 256 fp32
  static constexpr int EPI_WARPS = 8;
  static constexpr int STG_BUFS =  // per epilogue warp
      RESID_LN ? 2 : (RESID_F32 ? SRK_RESID_STG_BUFS : SRK_PAIR_STG_BUFS);
  static constexpr int STG_BYTES = 32 * 128;
  static constexpr int BAR_BYTES = 512;
  static constexpr int SMEM_BYTES =
      STAGES * STAGE_BYTES + EPI_WARPS * STG_BUFS * STG_BYTES + BAR_BYTES + 1024;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};

template <int EPI, int NP>
__global__ void __launch_bounds__(320, 1)
    gemm_bf16_tcgen05_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                                  const __grid_constant__ CUtensorMap tmB,
                                  const __grid_constant__ CUtensorMap tmC,
                                  const __grid_constant__ GemmLnArgs ln, int M, int N, int K,
                                  int rev) {
  using C = GemmPairCfg<EPI>;
  static_assert(NP == 1 || NP == 2, "one or two CTA pairs per cluster");
  constexpr int BN = C::BN;
  constexpr bool LN_IN = EPI == EPI_LN_BF16 || EPI == EPI_LN_GELU_BF16;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sStg = sB + C::STAGES * C::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + C::EPI_WARPS * C::STG_BUFS * C::STG_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* xbar = tempty + 2;  // EPI_RESID_LN: 1 per epilogue warp (x chunk loads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xbar + C::EPI_WARPS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int pr = static_cast<int>(rank >> 1);  // pair within the cluster
  const int cr = static_cast<int>(rank & 1);   // CTA within the pair
  const bool leader = cr == 0;
  const uint32_t lead_rank = rank & ~1u;
  const int pair = static_cast<int>(cluster_id_x());  // cluster index
  const int n_pairs = static_cast<int>(nclusters_x());
  const int m_tiles = (M + 2 * C::BM - 1) / (2 * C::BM);
  const int n_tiles = N / (BN * NP);  // cluster tiles along N
  const int num_tiles = m_tiles * n_tiles;
  // Tail split: when the last wave would leave at least half of the pairs
  // idle (num_tiles % n_pairs <= n_pairs / 2, e.g. the N = 1024 residual
  // GEMMs at C2: 388 tiles on 74 pairs), the tail tiles run as two 256 x 128
  // halves on twice as many pairs, so the last wave takes ~0.57 of a tile
  // (N = 128 MMAs) instead of a whole one. Generic epilogues only.
  constexpr bool kSplitOK = NP == 1 && SRK_TAIL_SPLIT &&
                            (EPI == EPI_BF16 || EPI == EPI_GELU_BF16 || EPI == EPI_RESID_F32 ||
                             EPI == EPI_F32);
  const int tail = num_tiles % n_pairs;
  const bool split = kSplitOK && tail > 0 && 2 * tail <= n_pairs;
  const int n_full = split ? num_tiles - tail : num_tiles;
  const int num_units = split ? n_full + 2 * tail : num_tiles;
  // unit -> (tile, half): half < 0 for a whole 256-column tile
  auto unit_tile = [&](int u, int& half) {
    if (u < n_full) {
      half = -1;
      return u;
    }
    half = (u - n_full) & 1;
    return n_full + ((u - n_full) >> 1);
  };

  const int nk = (K + C::BK - 1) / C::BK;
  // rev: walk the 256-row blocks from the last to the first, so the rows the
  // previous kernel wrote last (still in L2) are read first (serpentine order).
  auto m_block = [&](int tile) {
    const int mb = tile / n_tiles;
    return rev ? m_tiles - 1 - mb : mb;
  };
  if (threadIdx.x == 0) gemm_trace(0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmC);
    if constexpr (C::RESID_LN) tma_prefetch_desc(&ln.tm_xb);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 2);  // leader: own expect_tx arrival + the peer's arrival
      mbar_init(&empty[s], NP);  // one commit from every pair that reads the stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * C::EPI_WARPS);  // one per epilogue warp of both CTAs
    }
    if constexpr (C::RESID_LN)
      for (int b = 0; b < C::EPI_WARPS; ++b) mbar_init(&xbar[b], 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // inputs of the previous kernel (and its reads of our outputs) are done
  if (threadIdx.x == 0) gemm_trace(1);

  if (warp == 0) {
    if (lane == 0) {
#ifndef SRK_PAIR_APOL
#define SRK_PAIR_APOL 2
#endif
      const uint64_t pol_b = policy_evict_last();
      const uint64_t pol_a = SRK_PAIR_APOL == 0   ? policy_evict_first()
                             : SRK_PAIR_APOL == 1 ? policy_evict_normal()
                                                  : policy_evict_last();
      const uint32_t peer_full0 = mapa_shared(smem_u32(&full[0]), lead_rank);
      const uint16_t a_mask = static_cast<uint16_t>((1u << cr) | (1u << (cr + 2)));
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < num_units; u += n_pairs) {
        int half;
        const int tile = unit_tile(u, half);
        const int m0 = m_block(tile) * 2 * C::BM + cr * C::BM;
        // half tile: this CTA's 64 of the 128 columns (the 128-row box loads
        // 64 spare rows the N = 128 MMA does not read)
        const int n0 = ((tile % n_tiles) * NP + pr) * BN +
                       (half < 0 ? cr * (BN / 2) : half * (BN / 2) + cr * (BN / 4));
        if constexpr (C::RESID_LN) {
          // The epilogue reads this CTA's 128 x 256 fp32 slab of x after the
          // main loop: pull it into L2 now so those loads are L2 hits.
          const int xc = ((tile % n_tiles) * NP + pr) * BN;
          for (int rr = 0; rr < C::BM; rr += 32)
            for (int cc = 0; cc < BN; cc += 32) tma_prefetch_2d_l2(&tmC, xc + cc, m0 + rr);
        }
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (leader)
            mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
          else
            mbar_arrive_cluster(peer_full0 + stage * 8);
          if constexpr (NP == 1)
            tma_load_2d_pair(&tmA, &full[stage], sA + stage * C::A_BYTES, kb * C::BK, m0, pol_a);
          else if ((kb & 1) == pr)  // A is shared by both pairs: one multicast load
            tma_load_2d_pair_mc(&tmA, &full[stage], sA + stage * C::A_BYTES, kb * C::BK, m0,
                                a_mask, pol_a);
          tma_load_2d_pair(&tmB, &full[stage], sB + stage * C::B_BYTES, kb * C::BK, n0, pol_b);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(2 * C::BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      constexpr uint32_t idesc_half = idesc_bf16_f32(2 * C::BM, BN / 2);
      for (int u = pair; u < num_units; u += n_pairs, ++local) {
        int half;
        unit_tile(u, half);
        const uint32_t idu = half < 0 ? idesc : idesc_half;
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
          for (int k = 0; k < C::BK / 16; ++k)
            umma_bf16_pair(d_tmem, sw128_kmajor_desc(a_addr + k * 32),
                           sw128_kmajor_desc(b_addr + k * 32), idu, (kb | k) != 0 ? 1u : 0u);
          umma_commit_pair(&empty[stage], NP == 1 ? 0x3 : 0xF);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_pair(&tfull[acc], static_cast<uint16_t>(3u << (2 * pr)));
        if (local < 22) gemm_trace(2 + local);
      }
    }
    __syncwarp();
  } else {
    constexpr int CW = EpiOut<EPI>::CW;
    constexpr int SPAN = BN / 2;  // columns per epilogue warp
    const int quad = warp & 3;
    uint8_t* stg0 = sStg + (warp - 2) * C::STG_BUFS * C::STG_BYTES;
    const uint32_t tempty_leader = mapa_shared(smem_u32(&tempty[0]), lead_rank);
    const uint64_t pol_keep = policy_evict_last();
    int local = 0;
    int nstg = 0;  // staging chunks issued by this warp (buffer = nstg % STG_BUFS)
    uint32_t xph = 0;  // EPI_RESID_LN: parity of this warp's x-chunk barrier
    for (int u = pair; u < num_units; u += n_pairs, ++local) {
      int half;
      const int tile = unit_tile(u, half);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      const int m0 = m_block(tile) * 2 * C::BM + cr * C::BM;
      const int n0 = ((tile % n_tiles) * NP + pr) * BN + (half < 0 ? 0 : half * (BN / 2));
      // columns per epilogue warp (a half tile has 128 accumulator columns)
      const int span = half < 0 ? SPAN : SPAN / 2;
      const int col0 = ((warp - 2) >> 2) * span;
      const int r0 = m0 + quad * 32;
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + acc * BN;
      if constexpr (C::RESID_LN) {
        // One fp32 staging chunk F (x in, x + acc out) and one bf16 chunk Bb
        // per warp; x chunk c+1 is loaded (an L2 hit: the producer prefetched
        // the slab) as soon as chunk c's store has read F.
        uint8_t* F = stg0;
        uint8_t* Bb = stg0 + C::STG_BYTES;
        uint64_t* xb_bar = xbar + (warp - 2);
        if (r0 < M && lane == 0) {
          bulk_wait_read0();  // previous tile's stores have left F and Bb
          mbar_arrive_expect_tx(xb_bar, C::STG_BYTES);
          tma_load_2d(&tmC, xb_bar, F, n0 + col0, r0);
        }
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        if (r0 < M) {
          float s_mean = 0.f, s_m2 = 0.f;
#pragma unroll 1
          for (int c = 0; c < SPAN / 32; ++c) {
            __syncwarp();  // lane 0's buffer waits of the previous chunk come first
            uint32_t r[32];
            tmem_ld_32x32b_x32(t_row + col0 + 32 * c, r);
            mbar_wait(xb_bar, xph & 1u);
            xph ^= 1u;
            tmem_ld_wait();
            uint8_t* row = F + lane * 128;
            float v[32];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              uint4* qp = reinterpret_cast<uint4*>(row + ((k ^ (lane & 7)) * 16));
              const uint4 xv = *qp;
              v[4 * k + 0] = __uint_as_float(xv.x) + __uint_as_float(r[4 * k + 0]);
              v[4 * k + 1] = __uint_as_float(xv.y) + __uint_as_float(r[4 * k + 1]);
              v[4 * k + 2] = __uint_as_float(xv.z) + __uint_as_float(r[4 * k + 2]);
              v[4 * k + 3] = __uint_as_float(xv.w) + __uint_as_float(r[4 * k + 3]);
              *qp = make_uint4(__float_as_uint(v[4 * k]), __float_as_uint(v[4 * k + 1]),
                               __float_as_uint(v[4 * k + 2]), __float_as_uint(v[4 * k + 3]));
            }
            uint8_t* brow = Bb + lane * 128;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              *reinterpret_cast<uint4*>(brow + ((((c & 1) * 4 + k) ^ (lane & 7)) * 16)) =
                  make_uint4(pack_bf16x2(v[8 * k], v[8 * k + 1]),
                             pack_bf16x2(v[8 * k + 2], v[8 * k + 3]),
                             pack_bf16x2(v[8 * k + 4], v[8 * k + 5]),
                             pack_bf16x2(v[8 * k + 6], v[8 * k + 7]));
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmC, F, n0 + col0 + 32 * c, r0);
              bulk_commit();
              if (c & 1) {  // the bf16 copy is read next by QKV / W_in: keep it in L2
                tma_store_2d_hint(&ln.tm_xb, Bb, n0 + col0 + 32 * (c - 1), r0, pol_keep);
                bulk_commit();
              }
              if (c + 1 < SPAN / 32) {
                bulk_wait_read0();  // F (and Bb) have been read out
                mbar_arrive_expect_tx(xb_bar, C::STG_BYTES);
                tma_load_2d(&tmC, xb_bar, F, n0 + col0 + 32 * (c + 1), r0);
              }
            }
            // chunk mean / M2 (two-pass over registers, FFMA2), merged into the
            // running pair (Chan et al.); overlaps the next chunk's load
            uint64_t s2 = f32x2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < 32; j += 2) s2 = add_f32x2(s2, f32x2(v[j], v[j + 1]));
            float sa, sb;
            f32x2_split(s2, sa, sb);
            const float cm = (sa + sb) * (1.f / 32.f);
            const uint64_t ncm = f32x2(-cm, -cm);
            uint64_t q2 = f32x2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const uint64_t dv = add_f32x2(f32x2(v[j], v[j + 1]), ncm);
              q2 = fma_f32x2(dv, dv, q2);
            }
            float qa, qb;
            f32x2_split(q2, qa, qb);
            const float cq = qa + qb;
            if (c == 0) {
              s_mean = cm;
              s_m2 = cq;
            } else {
              const float na = 32.f * c, n = na + 32.f;
              const float dl = cm - s_mean;
              s_mean = fmaf(dl, 32.f / n, s_mean);
              s_m2 += cq + dl * dl * (na * 32.f / n);
            }
          }
          const int row = r0 + lane;
          if (row < M)
            ln.stats_out[static_cast<size_t>((n0 + col0) >> 7) * ln.ld + row] =
                make_float2(s_mean, s_m2);
        }
      } else {
        // EPI_LN_*: out = acc * rstd - mean * rstd * colsum (row stats per
        // lane); the partials are fetched before the accumulator wait.
        float ln_scale = 0.f, ln_shift = 0.f;
        float2 part[16];
        if constexpr (LN_IN) {
          const int row = r0 + lane;
          if (row < M) {
#pragma unroll
            for (int p = 0; p < 16; ++p)
              if (p < ln.n_parts) part[p] = ln.stats_in[static_cast<size_t>(p) * ln.ld + row];
          }
        }
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        if constexpr (LN_IN) {
          if (r0 + lane < M) {
            const int P = ln.n_parts;
            float mean = 0.f;
#pragma unroll
            for (int p = 0; p < 16; ++p)
              if (p < P) mean += part[p].x;
            mean /= static_cast<float>(P);
            const float cnt = static_cast<float>(K / P);
            float m2 = 0.f;
#pragma unroll
            for (int p = 0; p < 16; ++p)
              if (p < P) {
                const float dl = part[p].x - mean;
                m2 += fmaf(dl * dl, cnt, part[p].y);
              }
            ln_scale = 1.0f / sqrtf(m2 / static_cast<float>(K) + 1e-5f);
            ln_shift = -mean * ln_scale;
          }
        }
        if (r0 < M) {
#pragma unroll 1
          for (int c = col0; c < col0 + span; c += CW, ++nstg) {
            uint8_t* stg = stg0 + (nstg % C::STG_BUFS) * C::STG_BYTES;
            uint8_t* row_base = stg + lane * 128;
            if constexpr (C::RESID_F32 && SRK_RESID_RED == 2) {
              // 16x256b TMEM loads: four lanes own 32 contiguous bytes of a
              // row, so each REDG.ADD.F32x2 warp instruction covers 8 rows x
              // one full 32-byte sector
              if ((c - col0) % 64 != 0) continue;  // one pass per 64 columns
              const int t0 = lane & 3, t1 = lane >> 2;
#pragma unroll 1
              for (int hh = 0; hh < 2; ++hh) {
                uint32_t r[32];
                tmem_ld_16x256b_x8(tmem_base + (static_cast<uint32_t>(quad * 32 + hh * 16) << 16) +
                                       acc * BN + c, r);
                tmem_ld_wait();
                const int ra = r0 + hh * 16 + t1, rb = ra + 8;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const int col = n0 + c + 8 * i + 2 * t0;
                  if (ra < M)
                    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(
                                     ln.resid_out + static_cast<size_t>(ra) * ln.resid_ld + col),
                                 "f"(__uint_as_float(r[4 * i])), "f"(__uint_as_float(r[4 * i + 1]))
                                 : "memory");
                  if (rb < M)
                    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(
                                     ln.resid_out + static_cast<size_t>(rb) * ln.resid_ld + col),
                                 "f"(__uint_as_float(r[4 * i + 2])), "f"(__uint_as_float(r[4 * i + 3]))
                                 : "memory");
                }
              }
              continue;
            }
            if constexpr (C::RESID_F32 && SRK_RESID_RED == 1) {
              // x += acc straight from registers with vector reductions
              // (REDG.ADD.F32x4): no shared-memory staging, whose traffic
              // otherwise slows the operand-bound main loop of this GEMM.
              uint32_t r[32];
              tmem_ld_32x32b_x32(t_row + c, r);
              tmem_ld_wait();
              const int row = r0 + lane;
              if (row < M) {
                float* dst = ln.resid_out + static_cast<size_t>(row) * ln.resid_ld + n0 + c;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * q),
                               "f"(__uint_as_float(r[4 * q])), "f"(__uint_as_float(r[4 * q + 1])),
                               "f"(__uint_as_float(r[4 * q + 2])), "f"(__uint_as_float(r[4 * q + 3]))
                               : "memory");
              }
              continue;
            }
            if constexpr (EpiOut<EPI>::F32) {
              uint32_t r[32];
              tmem_ld_32x32b_x32(t_row + c, r);
              // The TMEM read overlaps the wait for this buffer's previous store.
              if (lane == 0) bulk_wait_read<C::STG_BUFS - 1>();
              __syncwarp();
              tmem_ld_wait();
#pragma unroll
              for (int k = 0; k < 8; ++k)
                *reinterpret_cast<uint4*>(row_base + ((k ^ (lane & 7)) * 16)) =
                    make_uint4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
            } else {
              uint32_t r[2][32];
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) tmem_ld_32x32b_x32(t_row + c + hh * 32, r[hh]);
              if (lane == 0) bulk_wait_read<C::STG_BUFS - 1>();
              __syncwarp();
              tmem_ld_wait();
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  float f[8];
                  if constexpr (LN_IN) {
                    const float4* cp =
                        reinterpret_cast<const float4*>(ln.colsum + n0 + c + hh * 32 + 8 * k);
                    const float4 c0v = __ldg(cp), c1v = __ldg(cp + 1);
                    const float csv[8] = {c0v.x, c0v.y, c0v.z, c0v.w, c1v.x, c1v.y, c1v.z, c1v.w};
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                      f[j] = fmaf(csv[j], ln_shift, __uint_as_float(r[hh][8 * k + j]) * ln_scale);
                  } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(r[hh][8 * k + j]);
                  }
                  if constexpr (EPI == EPI_GELU_BF16 || EPI == EPI_LN_GELU_BF16) {
#pragma unroll
                    for (int j = 0; j < 8; j += 2) gelu_erf_x2(f[j], f[j + 1]);
                  }
                  const int chunk = hh * 4 + k;
                  *reinterpret_cast<uint4*>(row_base + ((chunk ^ (lane & 7)) * 16)) =
                      make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                                 pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
                }
              }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              if constexpr (C::RESID_F32)  // x is re-read next by the LayerNorm
                tma_reduce_add_2d_hint(&tmC, stg, n0 + c, r0, pol_keep);
              else
                tma_store_2d(&tmC, stg, n0 + c, r0);
              bulk_commit();
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
      if (warp == 2 && lane == 0 && local < 38) gemm_trace(24 + local);
      if constexpr (EPI == EPI_RESID_F32_LN) {
        // Publish that this CTA's add-reductions into its 128-row block of x
        // are complete (one counter per block, N / 256 contributions); the
        // LayerNorm of the block runs in a concurrent kernel that waits for
        // the count (rowops.cu layer_norm_after_kernel), so it reads x from
        // L2 while the GEMM is still running. (Normalising the block in this
        // epilogue was measured 4x slower: the last contributor's 8 warps
        // took ~37 us per block and delayed their own tiles.) Opt-in: the
        // overlapped LayerNorm is slower than the separate pass at C2.
        if (lane == 0) {
          bulk_wait0();
          fence_proxy_async_global();
        }
        __syncwarp();
        named_bar_sync(1, 32 * C::EPI_WARPS);
        if (warp == 2 && lane == 0 && m0 < M) {  // blocks past M are never waited on
          __threadfence();
          atomicAdd(ln.ln_cnt + (m0 >> 7), 1u);
        }
      }
    }
    if (lane == 0) bulk_wait0();
  }

  pdl_trigger();  // this CTA's work is issued: the next kernel may start launching
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
  if (threadIdx.x == 0) gemm_trace(63);
}

}  // namespace srk
