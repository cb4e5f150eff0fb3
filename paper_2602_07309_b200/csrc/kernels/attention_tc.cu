// Segment-masked shared-prefix attention on 5th-generation tensor cores.
//
// Same semantics as kernels/attention.cu (reference kernels.cpp:51-95 with the
// multi-item mask of engine.cpp:147-184): query row r attends keys
// [prefix_begin, prefix_end) U [span_start, r]; softmax(q.k/sqrt(hd)) V.
//
// Persistent: one CTA per SM walks work items (128-row query tile x head);
// keys stream in blocks of 128 over each tile's two ranges (R1 = shared
// prefix, R2 = own segments). The block sequence is continuous across items,
// so the Q load and the O epilogue of one item overlap the next item's MMAs.
//   warp 0     TMA: Q (2 buffers, one per item parity), K_j / V_j 2-stage rings
//   warp 1     TMEM alloc + single-thread tcgen05.mma issuer:
//                S_j = Q K_j^T   SS-MMA -> TMEM S buffer (j & 1), 128 fp32 cols
//                O  += P_j V_j   TS-MMA: P_j from TMEM (bf16, aliased on the
//                                consumed S_j buffer), V_j from smem MN-major;
//                                O double-buffered by item parity
//   warps 2-9  softmax: two threads per query row (keys 0-63 / 64-127 of a
//              block): tcgen05.ld of the row slice, visibility bitmask (skipped
//              when the slice is fully visible), pair max exchange in smem,
//              P = ex2(..) as packed bf16x2 via tcgen05.st; per item epilogue
//              (deferred behind the next item's first block)
//              O / l -> bf16 -> HBM.
// Lazy rescaling (as FlashAttention-4): the exponent base only moves when the
// block max exceeds it by more than 2^8, so O is rescaled rarely and softmax
// of block j+1 overlaps PV_j and S_{j+2}. P <= 2^8 is exact enough in bf16 and
// the fp32 row sum uses the same base.
//
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,256+HD) O1 [384,384+HD).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <queue>
#include <vector>
#include <string>

#include "launch.h"
#include "ptx.cuh"

namespace srk {

namespace {

constexpr int kTM = 128;     // query rows per tile (UMMA M)
constexpr int kBK = 128;     // keys per block (UMMA N of S, K of PV)
constexpr int kBox = 16384;  // 128 rows x 128 B swizzle box
// Softmax threads per query row: each of the SL warps of a TMEM lane quadrant
// owns kBK / SL keys of every block. SL = 2 (8 softmax warps). SL = 4
// (-DSRK_ATTN_SLICES=4, 16 softmax warps, 576 threads) was built to hide more
// MUFU / TMEM latency but measured 2x slower at C2 (218k vs 112k cycles per
// CTA): the per-row overhead (masks, exchange, barrier, hand-off) is paid by
// twice as many threads, and at 576 threads ptxas caps registers at 96 (spills).
#ifndef SRK_ATTN_SLICES
#define SRK_ATTN_SLICES 2
#endif
template <int HD>
struct Slices {
  static constexpr int SL = HD == 128 ? SRK_ATTN_SLICES : 2;
  static constexpr int KEYS = kBK / SL;        // keys per softmax thread per block
  static constexpr int SOFTMAX = 128 * SL;     // softmax threads
  static constexpr int THREADS = 64 + SOFTMAX; // + TMA warp + MMA warp
  static constexpr int OCOLS = HD / SL;        // O columns per softmax thread
};
constexpr int kThreads = 320;  // attn_pp_kernel (kPPThreads) and helpers
constexpr float kRescaleLog2 = 8.0f;  // rescale O only when the max grows by > 2^8
// One exponential pair in kPolyEvery goes to the FMA pipe (0 = all on MUFU).
// Measured (tools/attn_trace.py, C2 layer): every 4th pair shortens the
// exponential phase ~1.3k -> ~1.05k cycles per block but the kernel slows
// 91.8k -> 100.2k cycles per CTA, so MUFU-only is the default.
#ifndef SRK_ATTN_POLY_EVERY
#define SRK_ATTN_POLY_EVERY 0
#endif
constexpr int kPolyEvery = SRK_ATTN_POLY_EVERY;
#ifndef SRK_ATTN_POLY3
#define SRK_ATTN_POLY3 1
#endif
#ifndef SRK_ATTN_S_WAIT
#define SRK_ATTN_S_WAIT 0
#endif
// Softmax loads the next block's S (when already complete) before this
// block's exponentials, so the TMEM read overlaps MUFU work. Measured slower
// at C2 (1.72 vs 1.51 ms per query; 1.92 when waiting for S_{g+1}), off.
#ifndef SRK_ATTN_PREFETCH
#define SRK_ATTN_PREFETCH 0
#endif
constexpr bool kPrefetchS = SRK_ATTN_PREFETCH != 0;
// Skip the exponentials of 32-key halves of a slice that no row of the warp
// sees (C2: 1.16 -> 1.05 x the needed exponentials). Measured slower (1.77 vs
// 1.54 ms per query: the warp-uniform branches inside the unrolled exp loop
// cost more than the MUFU work they save). Off.
// PV over only the K-steps a partial key block covers.
#ifndef SRK_ATTN_SHORT_PV
#define SRK_ATTN_SHORT_PV 1
#endif
constexpr bool kShortPV = SRK_ATTN_SHORT_PV != 0;
// S over only the (32-rounded) key columns a partial key block covers.
// Measured: no step gain, attention class 3-4% slower (3 rounds). Off.
#ifndef SRK_ATTN_SHORT_S
#define SRK_ATTN_SHORT_S 0
#endif
constexpr bool kShortS = SRK_ATTN_SHORT_S != 0;
// Exponentials before the pair max exchange for every block of an item but
// its first (recomputed when the max moves the base), so the max reduction
// and the exchange overlap the MUFU work. Bit-identical scores
// (tools/scores_dump.py), but measured slower at C2 (28.37k vs 28.53k pairs/s,
// attention class within noise, 3 interleaved rounds; 29.01k vs 29.23k with
// the max accumulated inside the exponential loop): off.
#ifndef SRK_ATTN_OPT_EXP
#define SRK_ATTN_OPT_EXP 0
#endif
constexpr bool kOptExp = SRK_ATTN_OPT_EXP != 0 && !kPrefetchS;
#ifndef SRK_ATTN_SKIP_HALVES
#define SRK_ATTN_SKIP_HALVES 0
#endif
constexpr bool kSkipHalves = SRK_ATTN_SKIP_HALVES != 0;

// Max of N floats with 8 independent FMNMX3 chains (latency-bound otherwise).
template <int N>
__device__ __forceinline__ float max_tree(const float (&s)[N]) {
  static_assert(N % 16 == 0, "max_tree");
  float m[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) m[c] = fmaxf(s[2 * c], s[2 * c + 1]);
#pragma unroll
  for (int i = 16; i < N; i += 16)
#pragma unroll
    for (int c = 0; c < 8; ++c) m[c] = fmax3f(m[c], s[i + 2 * c], s[i + 2 * c + 1]);
  return fmaxf(fmax3f(m[0], m[1], m[2]), fmax3f(fmaxf(m[3], m[4]), fmax3f(m[5], m[6], m[7]), -INFINITY));
}

template <int HD>
struct AttnCfg {
  static constexpr int NB = HD / 64;      // 64-wide boxes per row
  static constexpr int TILE = NB * kBox;  // Q / K / V tile bytes
  static constexpr int Q_OFF = 0;                 // 2 buffers
  static constexpr int K_OFF = Q_OFF + 2 * TILE;  // 2 stages
  static constexpr int V_OFF = K_OFF + 2 * TILE;  // 2 stages
  static constexpr int RED_OFF = V_OFF + 2 * TILE;
  // slots: max exchange by block parity (2 x SL x 128) + row sums (SL x 128)
  // + row sums handed to the epilogue warpgroup (2 items x SL x 128)
  static constexpr int LSUM_OFF = RED_OFF + 3 * Slices<HD>::SL * 128 * 4;
  static constexpr int BAR_OFF = LSUM_OFF + 2 * Slices<HD>::SL * 128 * 4;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static constexpr int O_COL = 2 * kBK;  // O buffer b at O_COL + b * 128
  static constexpr int TMEM_COLS = 512;
};

// Optional per-CTA timeline (clock64 stamps, 64 slots per CTA, first 256
// CTAs); enabled by attention_set_trace() for kernel tuning only.
__device__ unsigned long long* g_attn_trace = nullptr;
#ifndef SRK_TRACE_STRIDE
#define SRK_TRACE_STRIDE 64
#endif
#define SRK_TRACE(slot)                                                                      \
  do {                                                                                       \
    if (srk_trace != nullptr && blockIdx.x < 256)                                            \
      srk_trace[blockIdx.x * SRK_TRACE_STRIDE + (slot)] =                                    \
          static_cast<unsigned long long>(clock64());                                        \
  } while (0)
// Phase stamps inside the softmax of blocks 8..15 (tuning builds with
// -DSRK_ATTN_PHASES -DSRK_TRACE_STRIDE=256): slot 64 + 16 (g - 8) + phase.
#ifdef SRK_ATTN_PHASES
#define SRK_PHASE(cond, g, ph) \
  do {                         \
    if ((cond) && (g) >= 8 && (g) < 16) SRK_TRACE(64 + 16 * ((g) - 8) + (ph)); \
  } while (0)
#define SRK_ITEM(cond, li, k) \
  do {                        \
    if ((cond) && (li) < 8) SRK_TRACE(192 + 8 * (li) + (k)); \
  } while (0)
#else
#define SRK_PHASE(cond, g, ph) \
  do {                         \
  } while (0)
#define SRK_ITEM(cond, li, k) \
  do {                        \
  } while (0)
#endif

// Work-item order: head-major (item = h * n_tiles + tile, every tile of a head
// before the next head) or, with SRK_ATTN_ROWMAJOR, tile-major (the 8 heads
// of a tile on neighbouring CTAs, so a tile's Q/K/V rows are read from DRAM
// once and shared through L2 within the wave). Measured: within noise at C2
// (28.73k vs 28.66k pairs/s, 3 interleaved rounds); head-major stays.
#ifndef SRK_ATTN_ROWMAJOR
#define SRK_ATTN_ROWMAJOR 0
#endif
__device__ __forceinline__ int tile_of(int item, int n_tiles, int n_items) {
  if constexpr (SRK_ATTN_ROWMAJOR) return item / (n_items / n_tiles);
  return item % n_tiles;
}
__device__ __forceinline__ int head_of(int item, int n_tiles, int n_items) {
  if constexpr (SRK_ATTN_ROWMAJOR) return item % (n_items / n_tiles);
  return item / n_tiles;
}

// Walks the (item, block) sequence of one CTA.
struct Cursor {
  int li = -1;      // local item counter
  int item = 0;     // global work-item index
  int j = 0, nblk = 0, nb1 = 0;
  AttnTile t;
  int h = 0;
  bool valid = false;

  // Descriptor of the next item of this CTA, fetched one item ahead so the
  // global-load latency stays off the item boundary.
  AttnTile t_pre;
  int item_pre = -1, h_pre = 0;

  // Optional host-made work list (attention_work_lpt): item -> (tile, head),
  // tile < 0 = an empty slot; n_items is then the list's length.
  const int2* work = nullptr;

  __device__ AttnTile fetch(const AttnTile* tiles, int n_tiles, int n_items, int it, int& hh) const {
    if (work != nullptr) {
      const int2 w = work[it];
      hh = w.y;
      if (w.x < 0) return AttnTile{0, 0, 0, 0, 0, 0, 0, 0};  // no blocks: skipped
      return tiles[w.x];
    }
    hh = head_of(it, n_tiles, n_items);
    return tiles[tile_of(it, n_tiles, n_items)];
  }

  __device__ void load_item(const AttnTile* tiles, int n_tiles, int n_items, int item_) {
    item = item_;
    valid = item < n_items;
    if (!valid) return;
    int hh = 0, hp = 0;
    t = item == item_pre ? t_pre : fetch(tiles, n_tiles, n_items, item, hh);
    if (item == item_pre) hh = h_pre;
    const int nx = item + static_cast<int>(gridDim.x);
    if (nx < n_items) {
      t_pre = fetch(tiles, n_tiles, n_items, nx, hp);
      h_pre = hp;
      item_pre = nx;
    }
    h = hh;
    nb1 = (t.r1_end - t.r1_begin + kBK - 1) / kBK;
    nblk = nb1 + (t.r2_end - t.r2_begin + kBK - 1) / kBK;
    j = 0;
  }
  // First item with at least one block at or after `item_`.
  __device__ void next_item(const AttnTile* tiles, int n_tiles, int n_items, int item_) {
    do {
      ++li;
      load_item(tiles, n_tiles, n_items, item_);
      item_ += gridDim.x;
    } while (valid && nblk == 0);
  }
  __device__ void range(int& k0, int& kbeg, int& kend) const {
    if (j < nb1) {
      k0 = t.r1_begin + j * kBK;
      kbeg = t.r1_begin;
      kend = t.r1_end;
    } else {
      k0 = t.r2_begin + (j - nb1) * kBK;
      kbeg = t.r2_begin;
      kend = t.r2_end;
    }
  }
  // Advance one block; returns true when a new item started.
  __device__ bool advance(const AttnTile* tiles, int n_tiles, int n_items) {
    if (++j < nblk) return false;
    next_item(tiles, n_tiles, n_items, item + gridDim.x);
    return true;
  }
};

// EW: a dedicated epilogue warpgroup (warps 12-15) drains each item's O while
// the softmax warps (4-11) start the next item; setmaxnreg moves registers
// from the TMA / MMA / epilogue warpgroups to the two softmax warpgroups.
template <int HD, bool EW>
__global__ void __launch_bounds__(EW ? 512 : Slices<HD>::THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv,
                   const __grid_constant__ CUtensorMap tm_out, const RowSpan* __restrict__ spans,
                   const AttnTile* __restrict__ tiles, int n_tiles, __nv_bfloat16* __restrict__ out,
                   int n_heads, const int2* __restrict__ work, int n_work) {
  using C = AttnCfg<HD>;
  constexpr int SL = Slices<HD>::SL, KEYS = Slices<HD>::KEYS, OCOLS = Slices<HD>::OCOLS;
  constexpr int kSoftmaxThreads = Slices<HD>::SOFTMAX;
  static_assert(OCOLS % 32 == 0 && KEYS % 32 == 0, "slice layout");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // Align inside the shared window without leaving the shared address space.
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + C::Q_OFF;
  uint8_t* sK = smem + C::K_OFF;
  uint8_t* sV = smem + C::V_OFF;
  float* red = reinterpret_cast<float*>(smem + C::RED_OFF);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  uint64_t* q_full = bars + 0;    // [2] by item parity
  uint64_t* q_empty = bars + 2;   // [2]
  uint64_t* k_full = bars + 4;    // [2] by block parity
  uint64_t* k_empty = bars + 6;   // [2]
  uint64_t* v_full = bars + 8;    // [2]
  uint64_t* v_empty = bars + 10;  // [2]
  uint64_t* s_full = bars + 12;   // [2]
  uint64_t* p_full = bars + 14;   // [2]
  // [2] waited only before an O rescale or the item's epilogue; the phases no
  // one needs complete unwaited (compute-sanitizer synccheck: "missing wait")
  uint64_t* pv_done = bars + 16;
  uint64_t* o_empty = bars + 18;  // [2] by item parity
  uint64_t* o_full = bars + 20;   // [2] EW: last PV of the item done
  uint64_t* l_ready = bars + 22;  // [2] EW: the item's row sums are in smem
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);
  float* lsum_slot = reinterpret_cast<float*>(smem + C::LSUM_OFF);  // [2][SL][128]
  constexpr int SM_BASE = EW ? 4 : 2;  // first softmax warp

  const int n_items = work != nullptr ? n_work : n_tiles * n_heads;
  const int d = n_heads * HD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // read once: asm "memory" clobbers would otherwise reload it at every stamp
  unsigned long long* const srk_trace = g_attn_trace;
  if (threadIdx.x == 0) SRK_TRACE(0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], EW ? 4 : kSoftmaxThreads / 32);  // per storing warp
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], kSoftmaxThreads);
      mbar_init(&pv_done[s], 1);
      mbar_init(&o_empty[s], EW ? 128 : kSoftmaxThreads);
      mbar_init(&o_full[s], 1);
      mbar_init(&l_ready[s], kSoftmaxThreads);
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
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  // EW register split (2 x 128 x 184 + 2 x 128 x 72 = 65536): each role
  // branch re-budgets its warpgroup first, so ptxas compiles the softmax
  // code against 184 registers.
  auto regs_down = [] {
    if constexpr (EW) asm volatile("setmaxnreg.dec.sync.aligned.u32 72;" ::: "memory");
  };

#ifndef SRK_ATTN_SPLIT_KV
#define SRK_ATTN_SPLIT_KV 1
#endif
  constexpr bool kSplitKV = EW && SRK_ATTN_SPLIT_KV;
  if (warp == 0 || (kSplitKV && warp == 3)) {
    regs_down();
    // ------------------------------------------------------------- TMA
    // EW: warp 0 streams K, warp 3 streams V, so a K load never queues behind
    // the wait for a V stage (which frees only when PV of two blocks back has
    // run) — the K ring is what bounds how early S of the next block can go.
    const bool do_k = !kSplitKV || warp == 0, do_v = !kSplitKV || warp == 3;
    if (lane == 0) {
      const uint64_t keep = policy_evict_last();  // prefix K/V: re-read by every item tile
      Cursor c;
      c.work = work;
      c.next_item(tiles, n_tiles, n_items, blockIdx.x);
      int g = 0;
      while (c.valid) {
        if (!EW && c.j == 0) {  // EW: warp 2 loads Q, ahead of the K/V stream (!EW: one producer)
          const int qb = c.li & 1;
          mbar_wait(&q_empty[qb], ((c.li >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(&q_full[qb], C::TILE);
          for (int b = 0; b < C::NB; ++b)
            tma_load_2d(&tm_qkv, &q_full[qb], sQ + qb * C::TILE + b * kBox, c.h * HD + b * 64,
                        c.t.q_begin);
        }
        int k0, kb, ke;
        c.range(k0, kb, ke);
        const int st = g & 1;
        const uint32_t ph = ((g >> 1) & 1) ^ 1;
        if (do_k) {
          mbar_wait(&k_empty[st], ph);
          SRK_PHASE(true, g, 10);
          mbar_arrive_expect_tx(&k_full[st], C::TILE);
          for (int b = 0; b < C::NB; ++b)
            tma_load_2d_hint(&tm_qkv, &k_full[st], sK + st * C::TILE + b * kBox,
                             d + c.h * HD + b * 64, k0, keep);
        }
        if (do_v) {
          mbar_wait(&v_empty[st], ph);
          SRK_PHASE(true, g, 11);
          mbar_arrive_expect_tx(&v_full[st], C::TILE);
          for (int b = 0; b < C::NB; ++b)
            tma_load_2d_hint(&tm_qkv, &v_full[st], sV + st * C::TILE + b * kBox,
                             2 * d + c.h * HD + b * 64, k0, keep);
        }
        ++g;
        c.advance(tiles, n_tiles, n_items);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    regs_down();
    // ------------------------------------------------------------- MMA
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kTM, kBK);
      constexpr uint32_t idesc_pv = idesc_bf16_f32_bmn(kTM, HD);
      Cursor sc, pc;  // next block to issue S for / next block to issue PV for
      sc.work = work;
      sc.next_item(tiles, n_tiles, n_items, blockIdx.x);
      pc = sc;
      int gs = 0;  // global index of sc
      auto issue_s = [&]() {
        const int st = gs & 1;
        const int qb = sc.li & 1;
        if (sc.j == 0) mbar_wait(&q_full[qb], (sc.li >> 1) & 1);
        if (sc.j == 0) SRK_ITEM(true, sc.li, 4);
        mbar_wait(&k_full[st], (gs >> 1) & 1);
        tc_fence_after();
        SRK_PHASE(true, gs, 6);
        const uint32_t q_addr = smem_u32(sQ + qb * C::TILE);
        const uint32_t k_addr = smem_u32(sK + st * C::TILE);
        // a partial block computes only its ceil32(w) key columns (the rest of
        // the S buffer keeps stale values, all masked: keys >= ke are invisible)
        uint32_t ids = idesc_s;
        if constexpr (kShortS) {
          int k0, kb, ke;
          sc.range(k0, kb, ke);
          ids = idesc_bf16_f32(kTM, (min(kBK, ke - k0) + 31) & ~31);
        }
#pragma unroll
        for (int s = 0; s < HD / 16; ++s) {
          const uint32_t off = (s >> 2) * kBox + (s & 3) * 32;
          umma_bf16(tmem + st * kBK, sw128_kmajor_desc(q_addr + off),
                    sw128_kmajor_desc(k_addr + off), ids, s > 0 ? 1u : 0u);
        }
        umma_commit(&k_empty[st]);
        umma_commit(&s_full[st]);
        ++gs;
        sc.advance(tiles, n_tiles, n_items);
      };
      if (sc.valid) issue_s();
      if (sc.valid) issue_s();
      int g = 0;
      while (pc.valid) {
        const int st = g & 1;
        const uint32_t ph = (g >> 1) & 1;
        const int ob = pc.li & 1;
        if (pc.j == 0) mbar_wait(&o_empty[ob], ((pc.li >> 1) & 1) ^ 1);
        mbar_wait(&p_full[st], ph);
        SRK_PHASE(true, g, 8);
        mbar_wait(&v_full[st], ph);
        tc_fence_after();
        SRK_PHASE(true, g, 7);
        const uint32_t v_addr = smem_u32(sV + st * C::TILE);
        // a partial block (the tail of a key range) needs only ceil(w / 16)
        // K-steps of PV: its P columns past w are zero
        int nk = kBK / 16;
        if constexpr (kShortPV) {
          int k0, kb, ke;
          pc.range(k0, kb, ke);
          nk = (min(kBK, ke - k0) + 15) >> 4;
        }
#pragma unroll
        for (int s = 0; s < kBK / 16; ++s) {
          if (s >= nk) break;
          umma_bf16_ts(tmem + C::O_COL + ob * 128, tmem + st * kBK + s * 8,
                       sw128_mnmajor_desc(v_addr + s * 16 * 128, kBox, 1024), idesc_pv,
                       (pc.j > 0 || s > 0) ? 1u : 0u);
        }
        umma_commit(&v_empty[st]);
        umma_commit(&pv_done[st]);
        if (EW && pc.j + 1 == pc.nblk) umma_commit(&o_full[ob]);  // the item's O is final
        if (sc.valid) {
          // S_{g+2} reuses this TMEM buffer, whose P_g the PV_g just issued
          // reads. tcgen05.mma from one thread executes in issue order, so
          // S_{g+2} goes right behind PV_g (SRK_ATTN_S_WAIT=1: wait for PV_g's
          // commit first, one mbarrier round trip on the MMA chain per block).
#if SRK_ATTN_S_WAIT
          mbar_wait(&pv_done[st], ph);
#endif
          issue_s();
        }
        ++g;
        pc.advance(tiles, n_tiles, n_items);
      }
    }
    __syncwarp();
  } else if (EW && warp == 2) {
    regs_down();
    // ------------------------------------------------------ Q loads (EW)
    // Item i+1's Q loads as soon as the epilogue has released its buffer
    // (early in item i), instead of when the K/V stream reaches the item.
    if (lane == 0) {
      Cursor c;
      c.work = work;
      c.next_item(tiles, n_tiles, n_items, blockIdx.x);
      while (c.valid) {
        const int qb = c.li & 1;
        mbar_wait(&q_empty[qb], ((c.li >> 1) & 1) ^ 1);
        SRK_ITEM(true, c.li, 3);
        mbar_arrive_expect_tx(&q_full[qb], C::TILE);
        for (int b = 0; b < C::NB; ++b)
          tma_load_2d(&tm_qkv, &q_full[qb], sQ + qb * C::TILE + b * kBox, c.h * HD + b * 64,
                      c.t.q_begin);
        c.j = c.nblk - 1;
        c.advance(tiles, n_tiles, n_items);
      }
    }
    __syncwarp();
  } else if (EW && !kSplitKV && warp == 3) {
    regs_down();  // idle
  } else if (EW && warp >= 12) {
    regs_down();
    // ------------------------------------------ epilogue warpgroup (EW)
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    Cursor c;
    c.work = work;
    c.next_item(tiles, n_tiles, n_items, blockIdx.x);
    while (c.valid) {
      const int li = c.li, ob = li & 1, h = c.h, row0 = c.t.q_begin;
      const int row = row0 + r;
      const bool live = row < c.t.q_end;
      const uint32_t ph = (li >> 1) & 1;
      mbar_wait(&l_ready[ob], ph);
      SRK_ITEM(quad == 0 && lane == 0, li, 0);
      float lsum = 0.f;
#pragma unroll
      for (int k = 0; k < SL; ++k) lsum += lsum_slot[(ob * SL + k) * 128 + r];
      mbar_wait(&o_full[ob], ph);
      SRK_ITEM(quad == 0 && lane == 0, li, 1);
      tc_fence_after();
      const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
      // O / l -> bf16, staged in the item's Q buffer (every S of the item has
      // completed) and TMA-stored per 32-row slab; partially-live slabs
      // (request tails) store their live rows directly.
      uint8_t* qbuf = sQ + ob * C::TILE;
      const bool slab_live = __all_sync(0xffffffff, live);
#pragma unroll 1
      for (int cc = 0; cc < HD / 32; ++cc) {
        uint32_t v[32];
        const int col = cc * 32;
        tmem_ld_32x32b_x32(tmem + lane_off + C::O_COL + ob * 128 + col, v);
        tmem_ld_wait();
        uint4 pk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float* f = reinterpret_cast<const float*>(&v[q * 8]);
          pk[q] = make_uint4(pack_bf16x2(f[0] * inv, f[1] * inv), pack_bf16x2(f[2] * inv, f[3] * inv),
                             pack_bf16x2(f[4] * inv, f[5] * inv), pack_bf16x2(f[6] * inv, f[7] * inv));
        }
        if (slab_live) {
          uint8_t* rowp = qbuf + (col >> 6) * kBox + r * 128;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int chunk = ((col & 63) >> 3) + q;
            *reinterpret_cast<uint4*>(rowp + ((chunk ^ (r & 7)) * 16)) = pk[q];
          }
        } else if (live) {
          uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(row) * d + h * HD + col);
#pragma unroll
          for (int q = 0; q < 4; ++q) dst[q] = pk[q];
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      tc_fence_before();
      mbar_arrive(&o_empty[ob]);
      if (lane == 0) {
        if (slab_live)
          for (int b = 0; b < C::NB; ++b)
            tma_store_2d(&tm_out, qbuf + b * kBox + quad * 32 * 128, h * HD + b * 64,
                         row0 + quad * 32);
        bulk_commit();
        bulk_wait_read0();  // the Q buffer is reloaded for item li + 2
        mbar_arrive(&q_empty[ob]);
        SRK_ITEM(quad == 0, li, 2);
      }
      // next item (the epilogue walks items, not blocks)
      c.j = c.nblk - 1;
      c.advance(tiles, n_tiles, n_items);
    }
    if (lane == 0) bulk_wait0();
  } else if (warp >= SM_BASE && warp < SM_BASE + kSoftmaxThreads / 32) {
    if constexpr (EW) asm volatile("setmaxnreg.inc.sync.aligned.u32 184;" ::: "memory");
    // ---------------------------------------------------------- softmax
    const int quad = warp & 3;          // TMEM lane quadrant of this warp
    const int slice = (warp - SM_BASE) >> 2;  // keys [slice * KEYS, +KEYS) of every block
    const int r = quad * 32 + lane;     // tile row owned by this thread (with SL-1 partners)
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const float scale_log2 = 1.4426950408889634f * rsqrtf(static_cast<float>(HD));
    float* fin = red + 2 * SL * 128;
    const uint32_t qbar = 1 + quad, qbar_n = 32 * SL;  // the SL warps of this quadrant
    Cursor c;
    c.work = work;
    c.next_item(tiles, n_tiles, n_items, blockIdx.x);
    int g = 0;
    uint32_t nv[KEYS];  // S of the next block, prefetched (kPrefetchS)
    bool pre = false;
    // Row descriptor of the current item, fetched one item ahead.
    RowSpan sp_next = {0, 0, 0, 0};
    if (c.valid && c.t.q_begin + r < c.t.q_end) sp_next = spans[c.t.q_begin + r];
    // The O epilogue of item i is deferred until P of item i+1's first block
    // has been handed to the MMA warp, so the tensor core runs PV / S of the
    // next item while this warpgroup drains O (it used to sit idle for the
    // whole epilogue at every item boundary).
    struct Pending {
      bool on = false;
      int li = 0, h = 0, row0 = 0, g_last = 0;
      bool live = false;
      float l = 0.f;
    } pend;
    auto epilogue = [&](const Pending& e) {
      // Row sum over the slices (fixed order: identical in every slice), O / l
      // -> bf16 -> HBM.
      fin[slice * 128 + r] = e.l;
      named_bar_sync(qbar, qbar_n);
      float lsum = 0.f;
#pragma unroll
      for (int k = 0; k < SL; ++k) lsum += fin[k * 128 + r];
      mbar_wait(&pv_done[e.g_last & 1], (e.g_last >> 1) & 1);
      tc_fence_after();
      const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
      const int row = e.row0 + r;
      // Stage O (bf16) in this item's Q buffer — every S of the item has
      // completed — in the Q tile's own swizzled layout, then TMA-store each
      // fully-live 32-row slab; partially-live slabs (request tails) store
      // their live rows directly so neighbouring tiles are never touched.
      uint8_t* qbuf = sQ + (e.li & 1) * C::TILE;
      const bool slab_live = __all_sync(0xffffffff, e.live);
      constexpr int CW = OCOLS < 32 ? OCOLS : 32;  // columns per TMEM load
#pragma unroll 1
      for (int cc = 0; cc < OCOLS / CW; ++cc) {
        uint32_t v[32];
        const int col = slice * OCOLS + cc * CW;
        if constexpr (CW == 32)
          tmem_ld_32x32b_x32(tmem + lane_off + C::O_COL + (e.li & 1) * 128 + col, v);
        else
          tmem_ld_32x32b_x16(tmem + lane_off + C::O_COL + (e.li & 1) * 128 + col,
                             *reinterpret_cast<uint32_t(*)[16]>(v));
        tmem_ld_wait();
        uint4 pk[4];
#pragma unroll
        for (int q = 0; q < CW / 8; ++q) {
          const float* f = reinterpret_cast<const float*>(&v[q * 8]);
          pk[q] = make_uint4(pack_bf16x2(f[0] * inv, f[1] * inv), pack_bf16x2(f[2] * inv, f[3] * inv),
                             pack_bf16x2(f[4] * inv, f[5] * inv), pack_bf16x2(f[6] * inv, f[7] * inv));
        }
        if (slab_live) {
          uint8_t* rowp = qbuf + (col >> 6) * kBox + r * 128;
#pragma unroll
          for (int q = 0; q < CW / 8; ++q) {
            const int chunk = ((col & 63) >> 3) + q;
            *reinterpret_cast<uint4*>(rowp + ((chunk ^ (r & 7)) * 16)) = pk[q];
          }
        } else if (e.live) {
          uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(row) * d + e.h * HD + col);
#pragma unroll
          for (int q = 0; q < CW / 8; ++q) dst[q] = pk[q];
        }
      }
      fence_proxy_async_smem();
      // A 64-column box is written by 64 / OCOLS slices: they meet before the
      // first of them stores it.
      constexpr int SPB = 64 / OCOLS > 1 ? 64 / OCOLS : 1;  // slices per box
      if constexpr (SPB > 1) named_bar_sync(qbar, qbar_n);
      else __syncwarp();
      tc_fence_before();
      mbar_arrive(&o_empty[e.li & 1]);
      if (lane == 0) {
        // warp (quad, slice) with slice % SPB == 0 stores box slice / SPB of
        // rows [32 quad, +32)
        if (slab_live && slice % SPB == 0)
          tma_store_2d(&tm_out, qbuf + (slice / SPB) * kBox + quad * 32 * 128,
                       e.h * HD + (slice / SPB) * 64, e.row0 + quad * 32);
        bulk_commit();
        // Hand the Q buffer back once the store has read it: the producer
        // needs it for item li + 2, which may be the very next block (an
        // item of one block), so it cannot wait for a later hand-off.
        bulk_wait_read0();
        mbar_arrive(&q_empty[e.li & 1]);
      }
      if (warp == 2 && lane == 0 && e.li < 8) SRK_TRACE(56 + e.li);
    };
    while (c.valid) {
      const int c_row0 = c.t.q_begin;
      const int row = c_row0 + r;
      const bool live = row < c.t.q_end;
      const RowSpan sp = sp_next;
      // the next item's row descriptor, loaded while this item runs
      if (c.item_pre >= 0 && c.t_pre.q_begin + r < c.t_pre.q_end)
        sp_next = spans[c.t_pre.q_begin + r];
      float m_used = -INFINITY;  // exponent base (raw score units), shared by the pair
      float l = 0.f;             // this thread's partial row sum
      const int li = c.li, h = c.h;
      bool item_done = false;
      bool first = true;
      while (!item_done) {
        int k0, kb, ke;
        c.range(k0, kb, ke);
        const int sb = g & 1;
        const int kh = k0 + slice * KEYS;  // first key of this thread's slice
        float s[KEYS];
        if (pre) {
          // S of this block was loaded during the previous block's exponentials
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < KEYS; ++i) s[i] = __uint_as_float(nv[i]);
          pre = false;
        } else {
          mbar_wait(&s_full[sb], (g >> 1) & 1);
          if (warp == SM_BASE && lane == 0 && g < 24) SRK_TRACE(1 + g);
          if (c.j == 0) SRK_ITEM(warp == SM_BASE && lane == 0, c.li, 5);
          tc_fence_after();
          // all 32-column loads of the slice in flight, one wait
          uint32_t v[KEYS];
#pragma unroll
          for (int cc = 0; cc < KEYS / 32; ++cc)
            tmem_ld_32x32b_x32(tmem + lane_off + sb * kBK + slice * KEYS + cc * 32,
                               *reinterpret_cast<uint32_t(*)[32]>(&v[cc * 32]));
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < KEYS; ++i) s[i] = __uint_as_float(v[i]);
        }
        SRK_PHASE(warp == SM_BASE && lane == 0, g, 0);
        // Visible iff in [kb, ke) and in ([pb, pe) U [ss, row]).
        const int a_lo = max(kb, sp.prefix_begin), a_hi = min(ke, sp.prefix_end);
        const int b_lo = max(kb, sp.span_start), b_hi = min(ke, row + 1);
        const bool full = live && ((kh >= a_lo && kh + KEYS <= a_hi) ||
                                   (kh >= b_lo && kh + KEYS <= b_hi));
        float mx = -INFINITY;
        bool warp_empty = false;  // no visible key in this slice for any row of the warp
        // 32-key halves of the slice no row of the warp sees skip their
        // exponentials (C2: 1.16 -> 1.05 x the needed exponentials)
        bool half_on[KEYS / 32];
#pragma unroll
        for (int hf = 0; hf < KEYS / 32; ++hf) half_on[hf] = true;
        if (!__all_sync(0xffffffff, full)) {
          auto ivl = [&](int lo, int hi) -> uint64_t {
            lo = max(lo - kh, 0);
            hi = min(hi - kh, KEYS);
            if (!live || hi <= lo) return 0ull;
            const uint64_t upto_hi = hi >= 64 ? ~0ull : ((1ull << hi) - 1ull);
            return upto_hi & ~((1ull << lo) - 1ull);
          };
          const uint64_t vis = ivl(a_lo, a_hi) | ivl(b_lo, b_hi);
          warp_empty = !__any_sync(0xffffffff, vis != 0ull);
          if (!warp_empty) {
            const uint32_t v0 = static_cast<uint32_t>(vis), v1 = static_cast<uint32_t>(vis >> 32);
            if constexpr (kSkipHalves) {
              half_on[0] = __any_sync(0xffffffff, v0 != 0u);
              if constexpr (KEYS / 32 > 1) half_on[1] = __any_sync(0xffffffff, v1 != 0u);
            }
#pragma unroll
            for (int i = 0; i < KEYS; ++i) {
              const bool ok = ((i < 32 ? v0 : v1) >> (i & 31)) & 1u;
              s[i] = ok ? s[i] : -INFINITY;
            }
          }
        }
        // Pair max exchange (double-buffered by block parity). Only the two
        // warps sharing this row quadrant meet (named barrier 1 + quad, 64
        // threads), not all eight; the barrier also orders both halves' S
        // reads before either writes P over S (same TMEM lanes).
        float* slot = red + (g & 1) * SL * 128;
        auto exchange = [&](float m) -> float {
          slot[slice * 128 + r] = m;
          named_bar_sync(qbar, qbar_n);
#pragma unroll
          for (int k = 0; k < SL; ++k) m = fmaxf(m, slot[k * 128 + r]);
          return m;
        };
        // Every PV of this item so far used the old base: rescale O rows.
        auto rescale_o = [&](bool move, float m_new) {
          mbar_wait(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
          tc_fence_after();
          const float corr = move ? ex2_approx((m_used - m_new) * scale_log2) : 1.f;
          l *= corr;
#pragma unroll 1
          for (int cc = 0; cc < OCOLS / 32; ++cc) {
            uint32_t v[32];
            const uint32_t a = tmem + lane_off + C::O_COL + (li & 1) * 128 + slice * OCOLS + cc * 32;
            tmem_ld_32x32b_x32(a, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
            tmem_st_32x32b_x32(a, v);
          }
        };
        uint32_t pk[KEYS / 2];
        // P = 2^(s * scale - base) as packed bf16x2 + this thread's row sum.
        // Packed fp32x2 scale-subtract and row sums (FFMA2 / FADD2), MUFU
        // exponentials: the softmax is issue-bound (ncu: 41% issue active,
        // XU 19%), so the FMA-pipe exp2 emulation of earlier rounds cost
        // more issue slots than the MUFU time it saved.
        // with_max: the block's max accumulated inside the exponential loop
        // (4 FMNMX3 chains), so its ALU work issues between the MUFU ops.
        float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        auto exps = [&](bool with_max) -> float {
          if (warp_empty) {
#pragma unroll
            for (int i = 0; i < KEYS / 2; ++i) pk[i] = 0u;
            return 0.f;
          }
          const float base = m_used == -INFINITY ? 0.f : m_used * scale_log2;
          const uint64_t sc2 = f32x2(scale_log2, scale_log2), nb2 = f32x2(-base, -base);
          uint64_t acc0 = f32x2(0.f, 0.f), acc1 = acc0;
#pragma unroll
          for (int i = 0; i < KEYS; i += 2) {
            if (!half_on[i >> 5]) {  // warp-uniform: this half is masked for every row
              pk[i >> 1] = 0u;
              continue;
            }
            const uint64_t a2 = fma_f32x2(f32x2(s[i], s[i + 1]), sc2, nb2);
            if (with_max) mq[(i >> 1) & 3] = fmax3f(mq[(i >> 1) & 3], s[i], s[i + 1]);
            float p0, p1;
            if (kPolyEvery > 0 && (i >> 1) % kPolyEvery == kPolyEvery - 1) {
              // this pair on the FMA pipe: MUFU is the softmax's binding unit
              f32x2_split(SRK_ATTN_POLY3 ? ex2_poly3_x2(a2) : ex2_poly_x2(a2), p0, p1);
            } else {
              float a0, a1;
              f32x2_split(a2, a0, a1);
              p0 = ex2_approx(a0);
              p1 = ex2_approx(a1);
            }
            if (i & 2) acc1 = add_f32x2(acc1, f32x2(p0, p1));
            else acc0 = add_f32x2(acc0, f32x2(p0, p1));
            pk[i >> 1] = pack_bf16x2(p0, p1);
          }
          float r0, r1, r2, r3;
          f32x2_split(acc0, r0, r1);
          f32x2_split(acc1, r2, r3);
          return (r0 + r1) + (r2 + r3);
        };
        auto moves = [&](float m) {
          return m > m_used && (m_used == -INFINITY || (m - m_used) * scale_log2 > kRescaleLog2);
        };
        float rs;
        if (kOptExp && c.j > 0) {
          // Optimistic order (every block of an item but its first): the
          // exponentials run against the current base while this block's max
          // is still unknown, so the max reduction overlaps the MUFU work and
          // the pair exchange follows it. If the max moved the base (rare with
          // the 2^8 lazy-rescale margin), O is rescaled and the block's
          // exponentials are recomputed: P, the row sums and O are
          // bit-identical to the max-first order.
          SRK_PHASE(warp == SM_BASE && lane == 0, g, 1);
          rs = exps(true);
          mx = exchange(warp_empty ? -INFINITY : fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])));
          SRK_PHASE(warp == SM_BASE && lane == 0, g, 2);
          const bool move = moves(mx);
          if (__any_sync(0xffffffff, move)) {
            const float m_new = move ? mx : m_used;
            rescale_o(move, m_new);
            m_used = m_new;
            rs = exps(false);
          }
          SRK_PHASE(warp == SM_BASE && lane == 0, g, 3);
        } else {
          SRK_PHASE(warp == SM_BASE && lane == 0, g, 1);
          mx = exchange(warp_empty ? -INFINITY : max_tree<KEYS>(s));
          SRK_PHASE(warp == SM_BASE && lane == 0, g, 2);
          const bool move = moves(mx);
          const float m_new = move ? mx : m_used;
          if (c.j > 0 && __any_sync(0xffffffff, move)) rescale_o(move, m_new);
          m_used = m_new;
          SRK_PHASE(warp == SM_BASE && lane == 0, g, 3);
          if constexpr (kPrefetchS) {
            // Load the next block's S now, so the TMEM read (64 KB per block
            // over all softmax warps, ~1k cycles at the TMEM read rate) overlaps
            // this block's exponentials instead of following them.
            Cursor cn = c;
            cn.advance(tiles, n_tiles, n_items);
            // only when S_{g+1} is already complete (never stall this block on it)
            if (cn.valid && __all_sync(0xffffffff, mbar_test(&s_full[(g + 1) & 1], ((g + 1) >> 1) & 1))) {
              tc_fence_after();
#pragma unroll
              for (int cc = 0; cc < KEYS / 32; ++cc)
                tmem_ld_32x32b_x32(tmem + lane_off + ((g + 1) & 1) * kBK + slice * KEYS + cc * 32,
                                   *reinterpret_cast<uint32_t(*)[32]>(&nv[cc * 32]));
              pre = true;
            }
          }
          rs = exps(false);
        }
        l += rs;
        SRK_PHASE(warp == SM_BASE && lane == 0, g, 4);
        // P (bf16x2) over this slice's KEYS / 2 columns of the consumed S buffer
        // (columns of slices <= this one, already read: the quadrant barrier).
        if constexpr (KEYS == 64)
          tmem_st_32x32b_x32(tmem + lane_off + sb * kBK + slice * 32, pk);
        else
          tmem_st_32x32b_x16(tmem + lane_off + sb * kBK + slice * (KEYS / 2),
                             *reinterpret_cast<uint32_t(*)[16]>(pk));
        tmem_st_wait();
        SRK_PHASE(warp == SM_BASE && lane == 0, g, 5);
        SRK_PHASE(warp > SM_BASE && warp < SM_BASE + 4 && lane == 0, g, 12 + (warp - SM_BASE));
        SRK_PHASE(warp == SM_BASE + 4 && lane == 0, g, 9);
        tc_fence_before();
        mbar_arrive(&p_full[sb]);
        if (warp == SM_BASE && lane == 0 && g < 24) SRK_TRACE(32 + g);
        ++g;
        item_done = c.advance(tiles, n_tiles, n_items);
        if (first) {
          first = false;
          if constexpr (!EW) {
            // the previous item's epilogue, overlapping this item's MMAs.
            // Its pv_done wait is parity-safe: PV of block g_last + 2 (same
            // barrier) needs a P this warp has not produced yet.
            if (pend.on) epilogue(pend);
            pend.on = false;
          }
        }
      }
      if constexpr (EW) {
        // hand the row sums to the epilogue warpgroup and move on
        lsum_slot[((li & 1) * SL + slice) * 128 + r] = l;
        mbar_arrive(&l_ready[li & 1]);
        continue;
      }
      pend.on = true;
      pend.li = li;
      pend.h = h;
      pend.row0 = c_row0;
      pend.g_last = g - 1;
      pend.live = live;
      pend.l = l;
    }
    if (pend.on) epilogue(pend);
    if (lane == 0) bulk_wait0();  // O stores complete before exit
  }

  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
  if (threadIdx.x == 0) SRK_TRACE(29);
}

// The epilogue-warpgroup variant is the default (SRK_ATTN_EW=0 selects the
// 10-warp kernel whose softmax warps drain O themselves).
bool attn_use_ew() {
  static const bool ew = [] {
    const char* v = std::getenv("SRK_ATTN_EW");
    return Slices<128>::SL == 2 && (v == nullptr || std::atoi(v) != 0);
  }();
  return ew;
}

template <int HD, bool EW>
cudaError_t launch_tc_v(const CUtensorMap& tm, const RowSpan* spans, const AttnTile* tiles,
                        int n_tiles, __nv_bfloat16* out, int M, int n_heads, cudaStream_t stream,
                        const int2* work, int n_work) {
  using C = AttnCfg<HD>;
  auto kern = attn_tc_kernel<HD, EW>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // out [M x d] bf16, 64-column x 32-row boxes in the Q tile's swizzle.
  CUtensorMap tm_out;
  cudaError_t e = make_tmap_bf16_2d(&tm_out, out, M, static_cast<uint64_t>(n_heads) * HD, 32, 64);
  if (e != cudaSuccess) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  const int grid = attention_ctas(n_tiles, n_heads, dev);
  return launch_k(kern, dim3(grid), dim3(EW ? 512 : Slices<HD>::THREADS), C::SMEM, stream, tm,
                  tm_out, spans, tiles, n_tiles, out, n_heads, work, n_work);
}

template <int HD>
cudaError_t launch_tc(const CUtensorMap& tm, const RowSpan* spans, const AttnTile* tiles,
                      int n_tiles, __nv_bfloat16* out, int M, int n_heads, cudaStream_t stream,
                      const int2* work, int n_work) {
  if (Slices<HD>::SL == 2 && attn_use_ew())
    return launch_tc_v<HD, true>(tm, spans, tiles, n_tiles, out, M, n_heads, stream, work, n_work);
  return launch_tc_v<HD, false>(tm, spans, tiles, n_tiles, out, M, n_heads, stream, work, n_work);
}


// ----------------------------------------------------------------------------
// Ping-pong variant (opt-in, see attn_use_pp): two query tiles ("slots") in flight per CTA,
// as FlashAttention-4. Each slot has its own Q / K / V buffers, S/P and O
// TMEM regions and a 4-warp softmax group in which every thread owns one
// query row end to end (no cross-warp max exchange, no per-block CTA-wide
// barrier). The MMA warp issues whichever slot's next S or PV is ready, so
// the tensor core computes one slot's QK^T / PV while the other slot's
// softmax (and its item epilogue) runs.
//   warp 0 / 10  TMA producer of slot 0 / 1: K_j, V_j (single-stage per slot)
//   warp 1       TMEM alloc + event-driven tcgen05.mma issuer for both slots
//   warps 2-5    softmax + epilogue of slot 0 (rows = TMEM lanes, 128 threads)
//   warps 6-9    softmax + epilogue of slot 1
// The softmax group itself reloads its slot's Q once the item's O has been
// staged (in the Q buffer) and stored.
// TMEM (512 cols): S/P slot x at [128 x, +128), O slot x at [256 + 128 x, +HD).
constexpr int kPPThreads = 352;
// Key blocks of 64 rows (8 KB per 64-column box) so each slot gets a
// 2-stage K and V ring inside the smem budget (2 Q + 2 x 2 K + 2 x 2 V).
constexpr int kPB = 64;
constexpr int kPStages = 2;
constexpr int kKVBox = kPB * 128;

template <int HD>
struct PPCfg {
  static constexpr int NB = HD / 64;
  static constexpr int TILE = NB * kBox;      // Q tile (128 rows)
  static constexpr int KV_TILE = NB * kKVBox; // K / V block (64 rows)
  static constexpr int Q_OFF = 0;                                  // [slot]
  static constexpr int K_OFF = 2 * TILE;                           // [slot][stage]
  static constexpr int V_OFF = K_OFF + 2 * kPStages * KV_TILE;     // [slot][stage]
  static constexpr int BAR_OFF = V_OFF + 2 * kPStages * KV_TILE;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;
  static constexpr int O_COL = 256;
};

enum PPBar : int { PB_Q_FULL = 0, PB_K_FULL = 1, PB_K_EMPTY = 3, PB_V_FULL = 5,
                   PB_V_EMPTY = 7, PB_S_FULL = 9, PB_P_FULL = 10, PB_PV_DONE = 11, PB_N = 12 };

// One slot's (item, block) sequence: items first, first + stride, ...
struct SlotCursor {
  int item = 0, stride = 1, n_items = 0, n_tiles = 1;
  int j = 0, nblk = 0, nb1 = 0, h = 0;
  AttnTile t;
  bool valid = false;
  __device__ void init(const AttnTile* tiles, int n_tiles_, int n_items_, int first, int stride_) {
    n_tiles = n_tiles_;
    n_items = n_items_;
    stride = stride_;
    seek(tiles, first);
  }
  __device__ void seek(const AttnTile* tiles, int it) {
    for (;; it += stride) {
      item = it;
      valid = it < n_items;
      if (!valid) return;
      t = tiles[it % n_tiles];
      h = it / n_tiles;
      nb1 = (t.r1_end - t.r1_begin + kPB - 1) / kPB;
      nblk = nb1 + (t.r2_end - t.r2_begin + kPB - 1) / kPB;
      j = 0;
      if (nblk > 0) return;
    }
  }
  __device__ void range(int& k0, int& kbeg, int& kend) const {
    if (j < nb1) {
      k0 = t.r1_begin + j * kPB;
      kbeg = t.r1_begin;
      kend = t.r1_end;
    } else {
      k0 = t.r2_begin + (j - nb1) * kPB;
      kbeg = t.r2_begin;
      kend = t.r2_end;
    }
  }
  // Advance one block; true when the item finished.
  __device__ bool advance(const AttnTile* tiles) {
    if (++j < nblk) return false;
    seek(tiles, item + stride);
    return true;
  }
};

// Visible keys [lo, hi) (relative to the chunk start) as a 32-bit mask.
__device__ __forceinline__ uint32_t chunk_bits(int lo, int hi) {
  lo = max(lo, 0);
  hi = min(hi, 32);
  if (hi <= lo) return 0u;
  const uint32_t upto = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
  return upto & ~((1u << lo) - 1u);
}

template <int HD>
__global__ void __launch_bounds__(kPPThreads, 1)
    attn_pp_kernel(const __grid_constant__ CUtensorMap tm_qkv,
                   const __grid_constant__ CUtensorMap tm_kv,
                   const __grid_constant__ CUtensorMap tm_out, const RowSpan* __restrict__ spans,
                   const AttnTile* __restrict__ tiles, int n_tiles, __nv_bfloat16* __restrict__ out,
                   int n_heads) {
  using C = PPCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + C::Q_OFF;
  uint8_t* sK = smem + C::K_OFF;
  uint8_t* sV = smem + C::V_OFF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
  auto bar = [&](int x, int i) { return bars + x * PB_N + i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * PB_N);

  const int n_items = n_tiles * n_heads;
  const int d = n_heads * HD;
  const int G = static_cast<int>(gridDim.x);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // read once: asm "memory" clobbers would otherwise reload it at every stamp
  unsigned long long* const srk_trace = g_attn_trace;
  if (threadIdx.x == 0) SRK_TRACE(0);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_out);
    for (int x = 0; x < 2; ++x) {
      mbar_init(bar(x, PB_Q_FULL), 1);
      for (int st = 0; st < kPStages; ++st) {
        mbar_init(bar(x, PB_K_FULL + st), 1);
        mbar_init(bar(x, PB_K_EMPTY + st), 1);
        mbar_init(bar(x, PB_V_FULL + st), 1);
        mbar_init(bar(x, PB_V_EMPTY + st), 1);
      }
      mbar_init(bar(x, PB_S_FULL), 1);
      mbar_init(bar(x, PB_P_FULL), 128);
      mbar_init(bar(x, PB_PV_DONE), 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  if (warp == 0 || warp == 10) {
    // ------------------------------------------------ K / V of one slot
    const int x = warp == 0 ? 0 : 1;
    if (lane == 0) {
      const uint64_t keep = policy_evict_last();  // prefix K/V: re-read by every item tile
      SlotCursor c;
      c.init(tiles, n_tiles, n_items, blockIdx.x + x * G, 2 * G);
      for (int n = 0; c.valid; ++n) {
        int k0, kb, ke;
        c.range(k0, kb, ke);
        const int st = n & 1;
        const uint32_t ph = ((n >> 1) & 1) ^ 1;
        uint8_t* k_buf = sK + (x * kPStages + st) * C::KV_TILE;
        uint8_t* v_buf = sV + (x * kPStages + st) * C::KV_TILE;
        mbar_wait(bar(x, PB_K_EMPTY + st), ph);
        mbar_arrive_expect_tx(bar(x, PB_K_FULL + st), C::KV_TILE);
        for (int b = 0; b < C::NB; ++b)
          tma_load_2d_hint(&tm_kv, bar(x, PB_K_FULL + st), k_buf + b * kKVBox, d + c.h * HD + b * 64,
                           k0, keep);
        mbar_wait(bar(x, PB_V_EMPTY + st), ph);
        mbar_arrive_expect_tx(bar(x, PB_V_FULL + st), C::KV_TILE);
        for (int b = 0; b < C::NB; ++b)
          tma_load_2d_hint(&tm_kv, bar(x, PB_V_FULL + st), v_buf + b * kKVBox,
                           2 * d + c.h * HD + b * 64, k0, keep);
        c.advance(tiles);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA (both slots)
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kTM, kPB);
      constexpr uint32_t idesc_pv = idesc_bf16_f32_bmn(kTM, HD);
      SlotCursor c[2];
      int ns[2] = {0, 0}, np[2] = {0, 0}, nq[2] = {0, 0};
      bool want_s[2], s_free[2] = {true, true};
      for (int x = 0; x < 2; ++x) {
        c[x].init(tiles, n_tiles, n_items, blockIdx.x + x * G, 2 * G);
        want_s[x] = true;
      }
      while (c[0].valid || c[1].valid) {
#pragma unroll
        for (int x = 0; x < 2; ++x) {  // unrolled: per-slot state stays in registers
          if (!c[x].valid) continue;
          if (want_s[x]) {
            // S_x = Q_x K^T into the slot's S buffer, free once PV of the
            // previous block has read P out of it.
            if (!s_free[x]) {
              if (!mbar_test(bar(x, PB_PV_DONE), (np[x] - 1) & 1)) continue;
              s_free[x] = true;
            }
            if (c[x].j == 0 && !mbar_test(bar(x, PB_Q_FULL), nq[x] & 1)) continue;
            const int kst = ns[x] & 1;
            if (!mbar_test(bar(x, PB_K_FULL + kst), (ns[x] >> 1) & 1)) continue;
            tc_fence_after();
            if (c[x].j == 0) ++nq[x];
            const uint32_t q_addr = smem_u32(sQ + x * C::TILE);
            const uint32_t k_addr = smem_u32(sK + (x * kPStages + kst) * C::KV_TILE);
#pragma unroll
            for (int s = 0; s < HD / 16; ++s) {
              umma_bf16(tmem + x * kBK, sw128_kmajor_desc(q_addr + (s >> 2) * kBox + (s & 3) * 32),
                        sw128_kmajor_desc(k_addr + (s >> 2) * kKVBox + (s & 3) * 32), idesc_s,
                        s > 0 ? 1u : 0u);
            }
            umma_commit(bar(x, PB_K_EMPTY + kst));
            umma_commit(bar(x, PB_S_FULL));
            ++ns[x];
            want_s[x] = false;
          } else {
            // O_x += P_x V (P read from TMEM)
            const int vst = np[x] & 1;
            if (!mbar_test(bar(x, PB_P_FULL), np[x] & 1)) continue;
            if (!mbar_test(bar(x, PB_V_FULL + vst), (np[x] >> 1) & 1)) continue;
            tc_fence_after();
            const uint32_t v_addr = smem_u32(sV + (x * kPStages + vst) * C::KV_TILE);
#pragma unroll
            for (int s = 0; s < kPB / 16; ++s)
              umma_bf16_ts(tmem + C::O_COL + x * 128, tmem + x * kBK + s * 8,
                           sw128_mnmajor_desc(v_addr + s * 16 * 128, kKVBox, 1024), idesc_pv,
                           (c[x].j > 0 || s > 0) ? 1u : 0u);
            umma_commit(bar(x, PB_V_EMPTY + vst));
            umma_commit(bar(x, PB_PV_DONE));
            ++np[x];
            s_free[x] = false;
            want_s[x] = true;
            c[x].advance(tiles);
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ softmax + epilogue
    const int x = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // query row of the tile = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t t_s = tmem + lane_off + x * kBK;
    const uint32_t t_o = tmem + lane_off + C::O_COL + x * 128;
    uint8_t* qbuf = sQ + x * C::TILE;
    const bool elected = warp == 2 + 4 * x && lane == 0;
    const float scale_log2 = 1.4426950408889634f * rsqrtf(static_cast<float>(HD));
    SlotCursor c;
    c.init(tiles, n_tiles, n_items, blockIdx.x + x * G, 2 * G);
    auto load_q = [&]() {
      mbar_arrive_expect_tx(bar(x, PB_Q_FULL), C::TILE);
      for (int b = 0; b < C::NB; ++b)
        tma_load_2d(&tm_qkv, bar(x, PB_Q_FULL), qbuf + b * kBox, c.h * HD + b * 64, c.t.q_begin);
    };
    if (elected && c.valid) load_q();
    int g = 0;  // blocks of this slot so far
    while (c.valid) {
      const int row0 = c.t.q_begin;
      const int row = row0 + r;
      const bool live = row < c.t.q_end;
      const int h = c.h;
      RowSpan sp = {0, 0, 0, 0};
      if (live) sp = spans[row];
      float m_used = -INFINITY;  // exponent base (raw score units)
      float l = 0.f;
      bool item_done = false;
      while (!item_done) {
        int k0, kb, ke;
        c.range(k0, kb, ke);
        // visible keys of this row in the block, relative to k0
        const int a_lo = max(kb, sp.prefix_begin) - k0, a_hi = min(ke, sp.prefix_end) - k0;
        const int b_lo = max(kb, sp.span_start) - k0, b_hi = min(ke, row + 1) - k0;
        const bool full = live && ((a_lo <= 0 && a_hi >= kPB) || (b_lo <= 0 && b_hi >= kPB));
        const bool all_full = __all_sync(0xffffffff, full);
        mbar_wait(bar(x, PB_S_FULL), g & 1);
        if (warp == 2 && lane == 0 && g < 24) SRK_TRACE(40 + g);
        tc_fence_after();
        // The whole 128-key row of S in registers: one TMEM round trip.
        uint32_t v[kPB];
#pragma unroll
        for (int cc = 0; cc < kPB / 32; ++cc)
          tmem_ld_32x32b_x32(t_s + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&v[cc * 32]));
        uint32_t bits[kPB / 32];
#pragma unroll
        for (int cc = 0; cc < kPB / 32; ++cc)
          bits[cc] = all_full ? 0xffffffffu
                              : (live ? (chunk_bits(a_lo - 32 * cc, a_hi - 32 * cc) |
                                         chunk_bits(b_lo - 32 * cc, b_hi - 32 * cc))
                                      : 0u);
        tmem_ld_wait();
        float ma = -INFINITY, mb = -INFINITY;
        if (all_full) {
#pragma unroll
          for (int i = 0; i < kPB; i += 4) {
            ma = fmax3f(ma, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
            mb = fmax3f(mb, __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
          }
        } else {
#pragma unroll
          for (int i = 0; i < kPB; i += 2) {
            if (!((bits[i >> 5] >> (i & 31)) & 1u)) v[i] = __float_as_uint(-INFINITY);
            if (!((bits[i >> 5] >> ((i + 1) & 31)) & 1u)) v[i + 1] = __float_as_uint(-INFINITY);
            if (i & 2) mb = fmax3f(mb, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
            else ma = fmax3f(ma, __uint_as_float(v[i]), __uint_as_float(v[i + 1]));
          }
        }
        const float mx = fmaxf(ma, mb);
        // Lazy rescale (FlashAttention-4): move the base only when the max
        // grows by more than 2^8; O is rescaled in TMEM by its own row's thread.
        const bool move =
            mx > m_used && (m_used == -INFINITY || (mx - m_used) * scale_log2 > kRescaleLog2);
        const float m_new = move ? mx : m_used;
        if (c.j > 0 && __any_sync(0xffffffff, move)) {
          mbar_wait(bar(x, PB_PV_DONE), (g - 1) & 1);  // every PV so far used the old base
          tc_fence_after();
          const float corr = move ? ex2_approx((m_used - m_new) * scale_log2) : 1.f;
          l *= corr;
#pragma unroll 1
          for (int cc = 0; cc < HD / 32; ++cc) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(t_o + cc * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
            tmem_st_32x32b_x32(t_o + cc * 32, o);
          }
        }
        m_used = m_new;
        const float base = m_used == -INFINITY ? 0.f : m_used * scale_log2;
        const uint64_t sc2 = f32x2(scale_log2, scale_log2), nb2 = f32x2(-base, -base);
        uint64_t acc0 = f32x2(0.f, 0.f), acc1 = acc0;
        // P = 2^(s * scale - base) as bf16x2 over the consumed S columns
        // (keys 32 cc .. 32 cc + 31 -> columns [16 cc, 16 cc + 16)), packed in
        // place into v[32 cc .. 32 cc + 15]; masked keys hold -inf -> 0.
#pragma unroll
        for (int cc = 0; cc < kPB / 32; ++cc) {
          uint32_t* w = &v[32 * cc];
          if (!__any_sync(0xffffffff, bits[cc] != 0u)) {
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i] = 0u;
          } else {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              float a0, a1;
              f32x2_split(fma_f32x2(f32x2(__uint_as_float(w[i]), __uint_as_float(w[i + 1])), sc2,
                                    nb2),
                          a0, a1);
              const float p0 = ex2_approx(a0);
              const float p1 = ex2_approx(a1);
              if (i & 2) acc1 = add_f32x2(acc1, f32x2(p0, p1));
              else acc0 = add_f32x2(acc0, f32x2(p0, p1));
              w[i >> 1] = pack_bf16x2(p0, p1);
            }
          }
          tmem_st_32x32b_x16(t_s + cc * 16, *reinterpret_cast<uint32_t(*)[16]>(w));
        }
        float r0, r1, r2, r3;
        f32x2_split(acc0, r0, r1);
        f32x2_split(acc1, r2, r3);
        l += (r0 + r1) + (r2 + r3);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(bar(x, PB_P_FULL));
        if (warp == 2 && lane == 0 && g < 24) SRK_TRACE(1 + g);
        ++g;
        item_done = c.advance(tiles);
      }
      // ---- item epilogue: O / l -> bf16, staged in this slot's Q buffer
      // (every S of the item has completed), TMA-stored per 32-row slab;
      // partially-live slabs (request tails) store their live rows directly.
      mbar_wait(bar(x, PB_PV_DONE), (g - 1) & 1);
      tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const bool slab_live = __all_sync(0xffffffff, live);
#pragma unroll 1
      for (int cc = 0; cc < HD / 32; ++cc) {
        uint32_t v[32];
        const int col = cc * 32;
        tmem_ld_32x32b_x32(t_o + col, v);
        tmem_ld_wait();
        uint4 pk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float* f = reinterpret_cast<const float*>(&v[q * 8]);
          pk[q] = make_uint4(pack_bf16x2(f[0] * inv, f[1] * inv), pack_bf16x2(f[2] * inv, f[3] * inv),
                             pack_bf16x2(f[4] * inv, f[5] * inv), pack_bf16x2(f[6] * inv, f[7] * inv));
        }
        if (slab_live) {
          uint8_t* rowp = qbuf + (col >> 6) * kBox + r * 128;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int chunk = ((col & 63) >> 3) + q;
            *reinterpret_cast<uint4*>(rowp + ((chunk ^ (r & 7)) * 16)) = pk[q];
          }
        } else if (live) {
          uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(row) * d + h * HD + col);
#pragma unroll
          for (int q = 0; q < 4; ++q) dst[q] = pk[q];
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (slab_live)
          for (int b = 0; b < C::NB; ++b)
            tma_store_2d(&tm_out, qbuf + b * kBox + quad * 32 * 128, h * HD + b * 64, row0 + quad * 32);
        bulk_commit();
        bulk_wait_read0();  // the Q buffer is reloaded next
      }
      tc_fence_before();
      named_bar_sync(2 + x, 128);  // all four slabs have left the Q buffer
      if (elected && c.valid) load_q();
      if (warp == 2 && lane == 0 && g < 256) SRK_TRACE(30);
    }
    if (lane == 0) bulk_wait0();  // O stores complete before exit
  }

  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
  if (threadIdx.x == 0) SRK_TRACE(29);
}

template <int HD>
cudaError_t launch_pp(const CUtensorMap& tm, const void* qkv, const RowSpan* spans,
                      const AttnTile* tiles, int n_tiles, __nv_bfloat16* out, int M, int n_heads,
                      cudaStream_t stream) {
  using C = PPCfg<HD>;
  auto kern = attn_pp_kernel<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  CUtensorMap tm_out, tm_kv;
  cudaError_t e = make_tmap_bf16_2d(&tm_out, out, M, static_cast<uint64_t>(n_heads) * HD, 32, 64);
  if (e != cudaSuccess) return e;
  // K / V blocks of kPB rows; rows past M are never visible (masked) and the
  // packed buffer is padded, but keep the map exact: clip at M.
  e = make_tmap_bf16_2d(&tm_kv, qkv, M, static_cast<uint64_t>(3 * n_heads) * HD, kPB, 64);
  if (e != cudaSuccess) return e;
  int dev = 0;
  cudaGetDevice(&dev);
  const int items = n_tiles * n_heads;
  // two items in flight per CTA
  const int want = (items + 1) / 2;
  const int grid = want < num_sms(dev) ? want : num_sms(dev);
  return launch_k(kern, dim3(grid), dim3(kPPThreads), C::SMEM, stream, tm, tm_kv, tm_out, spans,
                  tiles, n_tiles, out, n_heads);
}

// Opt-in (SRK_ATTN=pp). Measured on B200 at C2 (tools/attn_pp_trace.py):
// with 128-key blocks and one K/V stage per slot, 132k cycles per CTA vs 112k
// for attn_tc_kernel; with 64-key blocks and 2-stage K/V rings per slot (this
// version) 157-162k: the softmax of a 64-key block takes ~1.2k cycles per
// slot, but each slot then waits ~2.7k cycles for its next S (PV -> S
// dependency through the S/P buffer plus two commit -> mbarrier -> poll hops
// per block), so the two slots still do not hide each other.
bool attn_use_pp() {
  static const bool pp = [] {
    const char* v = std::getenv("SRK_ATTN");
    return v != nullptr && std::string(v) == "pp";
  }();
  return pp;
}
}  // namespace

cudaError_t attention_fa_set_trace(unsigned long long* dev_buf);
cudaError_t attention_eo_set_trace(unsigned long long* dev_buf);
cudaError_t attention_set_trace(unsigned long long* dev_buf) {
  cudaError_t e = attention_fa_set_trace(dev_buf);
  if (e != cudaSuccess) return e;
  e = attention_eo_set_trace(dev_buf);
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(g_attn_trace, &dev_buf, sizeof(dev_buf));
}

int attention_tile_rows(int head_dim) { return head_dim >= 64 ? kTM : 64; }

// attention_fa.cu: two query tiles per CTA (head 128, opt-in SRK_ATTN=fa).
bool attn_use_fa();
// attention_eo.cu: softmax warps own alternate key blocks (head 128, SRK_ATTN=eo).
bool attn_use_eo();
cudaError_t attention_eo(const CUtensorMap& tm_qkv, const RowSpan* spans, const AttnTile* tiles,
                         int n_tiles, __nv_bfloat16* out, int n_heads, cudaStream_t stream);
cudaError_t attention_fa(const CUtensorMap& tm_qkv, const RowSpan* spans, const AttnTile* tiles,
                         int n_tiles, __nv_bfloat16* out, int n_heads, cudaStream_t stream);

int attention_ctas(int n_tiles, int n_heads, int device) {
  const int items = n_tiles * n_heads;
  return items < num_sms(device) ? items : num_sms(device);
}

void attention_work_lpt(const AttnTile* tiles, int n_tiles, int n_heads, int ctas,
                        std::vector<int2>& out) {
  // cost of a (tile, head) item in key blocks, + ~1/2 block of per-item work
  // (Q load, O epilogue hand-off); identical for every head of a tile
  std::vector<std::pair<double, int>> items;  // (cost, tile)
  items.reserve(static_cast<size_t>(n_tiles));
  for (int t = 0; t < n_tiles; ++t) {
    const AttnTile& a = tiles[t];
    const int nb = (a.r1_end - a.r1_begin + kBK - 1) / kBK + (a.r2_end - a.r2_begin + kBK - 1) / kBK;
    items.push_back({nb + 0.5, t});
  }
  std::vector<int> seq;
  for (int t = 0; t < n_tiles; ++t) seq.push_back(t);
  std::stable_sort(seq.begin(), seq.end(),
                   [&](int a, int b) { return items[a].first > items[b].first; });
  std::vector<std::vector<int2>> lists(static_cast<size_t>(ctas));
  // at most `cap` items per CTA, so the list length (a kernel argument baked
  // into captured graphs) depends only on (n_tiles, n_heads, ctas)
  const size_t n_items = static_cast<size_t>(n_tiles) * n_heads;
  const size_t cap = (n_items + ctas - 1) / ctas + 1;
  // min-load CTA first (ties: lowest index), items heaviest first, heads of a
  // tile consecutively so concurrent CTAs share the tile's rows in L2
  std::priority_queue<std::pair<double, int>, std::vector<std::pair<double, int>>,
                      std::greater<std::pair<double, int>>>
      heap;
  for (int c = 0; c < ctas; ++c) heap.push({0.0, c});
  for (int t : seq)
    for (int h = 0; h < n_heads; ++h) {
      auto [l, c] = heap.top();
      heap.pop();
      lists[c].push_back(make_int2(t, h));
      if (lists[c].size() < cap) heap.push({l + items[t].first, c});
    }
  out.assign(cap * static_cast<size_t>(ctas), make_int2(-1, 0));
  for (int c = 0; c < ctas; ++c)
    for (size_t k = 0; k < lists[c].size(); ++k) out[k * ctas + c] = lists[c][k];
}

cudaError_t attention_tc(const CUtensorMap& tm_qkv, const void* qkv, const RowSpan* spans,
                         const AttnTile* tiles, int n_tiles, __nv_bfloat16* out, int M,
                         int n_heads, int head_dim, cudaStream_t stream, const int2* work,
                         int n_work) {
  if (n_tiles <= 0) return cudaSuccess;
  if (head_dim == 128 && attn_use_fa())
    return attention_fa(tm_qkv, spans, tiles, n_tiles, out, n_heads, stream);
  if (head_dim == 128 && attn_use_eo())
    return attention_eo(tm_qkv, spans, tiles, n_tiles, out, n_heads, stream);
  // SRK_ATTN=pp selects the two-slot ping-pong kernel (A/B runs).
  const bool pp = attn_use_pp();
  switch (head_dim) {
    case 64:
      return pp ? launch_pp<64>(tm_qkv, qkv, spans, tiles, n_tiles, out, M, n_heads, stream)
                : launch_tc<64>(tm_qkv, spans, tiles, n_tiles, out, M, n_heads, stream, work,
                                n_work);
    case 128:
      return pp ? launch_pp<128>(tm_qkv, qkv, spans, tiles, n_tiles, out, M, n_heads, stream)
                : launch_tc<128>(tm_qkv, spans, tiles, n_tiles, out, M, n_heads, stream, work,
                                 n_work);
  }
  return cudaErrorInvalidValue;
}

}  // namespace srk
