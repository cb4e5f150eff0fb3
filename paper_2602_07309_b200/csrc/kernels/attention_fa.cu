// Segment-masked shared-prefix attention, two query tiles per CTA (head 128).
//
// Same semantics as kernels/attention_tc.cu and kernels/attention.cu
// (reference kernels.cpp:51-95 with the multi-item mask of engine.cpp:147-184):
// query row r attends keys [prefix_begin, prefix_end) U [span_start, r];
// softmax(q.k / sqrt(hd)) V.
//
// Work item = (pair of consecutive 128-row query tiles, head). The two tiles
// ("slots" 0 and 1) run in ping-pong as in FlashAttention-4: while one slot's
// softmax warpgroup turns S into P, the tensor core computes the other slot's
// PV and next S, so neither the MUFU pipe nor the tensor pipe waits on a
// lock-stepped partner. Both slots read one K/V stream: a shared-prefix block
// both tiles need is loaded once and consumed by both (the prefix is 2 of the
// ~4 key blocks of a C2 tile).
//
// Key blocks of a tile: its prefix range in 128-key blocks, then its own
// segment range aligned on the tile itself — a diagonal block [q_begin,
// q_end) and, walking back from q_begin, the earlier keys of the tile's first
// item (the last of them only as wide as needed, rounded up to 32 keys). At
// C2 (96-token items) that is 128 + {0, 32, 64} own keys per tile instead of
// 1-2 full blocks from the first item's start.
//
// Rounds: round i issues, for each slot with an i-th block, PV of the slot's
// previous block and then S of its i-th block. PVs therefore retire loads in
// load order, which keeps the K and V rings deadlock-free at depth 2.
//   warp 0      TMA producer: K blocks          warp 3  TMA producer: V blocks
//   warp 1      TMEM alloc + single-thread tcgen05.mma issuer
//   warp 2      TMA producer: Q tiles (ring of kQB buffers)
//   warps 4-7   softmax of slot 0: one thread per query row, all 128 keys of a
//               block in registers, P (bf16x2) written over S in TMEM
//   warps 8-11  softmax of slot 1
//   warps 12-15 epilogue: O / l -> bf16 -> HBM per tile, releases O in TMEM
// TMEM (512 cols): S/P slot x at [128 x, +128), O slot x at [256 + 128 x, +128).
// Lazy rescale (FlashAttention-4): the exponent base moves only when the block
// max exceeds it by more than 2^8.
#include <cuda_bf16.h>

#include <cstdlib>

#include "attn_blocks.cuh"
#include "launch.h"
#include "ptx.cuh"

namespace srk {

namespace {

constexpr int kFHD = 128;            // head dim
constexpr int kFTM = 128;            // query rows per tile
using attn::kFBK;                     // keys per block (max)
using attn::FaTile;
using attn::fa_bits;
constexpr int kFBox = 16384;         // 128 rows x 128 B (64 bf16) swizzle box
constexpr int kFTile = 2 * kFBox;    // Q / K / V tile (128 rows x 128 dims)
#ifndef SRK_FA_QBUFS
#define SRK_FA_QBUFS 2
#endif
#ifndef SRK_FA_KSTAGES
#define SRK_FA_KSTAGES 2
#endif
#ifndef SRK_FA_VSTAGES
#define SRK_FA_VSTAGES 3
#endif
constexpr int kQB = SRK_FA_QBUFS, kKS = SRK_FA_KSTAGES, kVS = SRK_FA_VSTAGES;
constexpr int kFThreads = 512;
// One exponential pair in kFPoly goes to the FMA pipe (Cody-Waite + degree-4
// polynomial, ptx.cuh ex2_poly_x2); 0 = all on MUFU.
#ifndef SRK_FA_POLY
#define SRK_FA_POLY 0
#endif
constexpr int kFPoly = SRK_FA_POLY;
constexpr float kFRescaleLog2 = 8.0f;

constexpr int F_Q_OFF = 0;
constexpr int F_K_OFF = F_Q_OFF + kQB * kFTile;
constexpr int F_V_OFF = F_K_OFF + kKS * kFTile;
constexpr int F_LSUM_OFF = F_V_OFF + kVS * kFTile;     // [2 slots][128] row sums
constexpr int F_BAR_OFF = F_LSUM_OFF + 2 * 128 * 4;
constexpr int F_SMEM = F_BAR_OFF + 256 + 1024;         // + alignment slack
static_assert(F_SMEM <= 232448, "attention_fa: shared memory budget");
constexpr uint32_t F_S_COL = 0, F_O_COL = 256;

// Optional per-CTA clock64 timeline (256 slots per CTA, tuning only; set by
// attention_set_trace): MMA 6e+{0 wait P, 1 got P, 2 got V, 3 PV issued,
// 4 got K, 5 S issued} for the first 16 (round, slot) events; softmax 96 + 48x + 2b + {0 S seen, 1 P
// handed}; epilogue 192 + 4e + {0 l, 1 O, 2 stored}; 224 start, 225 end.
__device__ unsigned long long* g_fa_trace = nullptr;
#define FA_TRACE(slot)                                                                     \
  do {                                                                                     \
    if (fa_trace != nullptr && (slot) < 256)                                               \
      fa_trace[blockIdx.x * 256 + (slot)] = static_cast<unsigned long long>(clock64());    \
  } while (0)

// One work item: (tile pair, head).
struct FaWork {
  FaTile s[2];
  bool two = false;
  int nsh = 0;     // leading rounds whose block both slots share (prefix)
  int rounds = 0;
  int h = 0;
  __device__ void load(const AttnTile* tiles, int n_tiles, int n_pairs, int item) {
    h = item / n_pairs;
    const int p = item - h * n_pairs;
    s[0].set(tiles[2 * p]);
    two = 2 * p + 1 < n_tiles;
    if (two) s[1].set(tiles[2 * p + 1]);
    else s[1].n = 0;
    nsh = 0;
    if (two && s[0].t.r1_begin == s[1].t.r1_begin && s[0].t.r1_end == s[1].t.r1_end)
      nsh = s[0].nb1;
    rounds = max(s[0].n, s[1].n);
  }
};

__global__ void __launch_bounds__(kFThreads, 1)
    attn_fa_kernel(const __grid_constant__ CUtensorMap tm_qkv, const RowSpan* __restrict__ spans,
                   const AttnTile* __restrict__ tiles, int n_tiles, __nv_bfloat16* __restrict__ out,
                   int n_heads) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + F_Q_OFF;
  uint8_t* sK = smem + F_K_OFF;
  uint8_t* sV = smem + F_V_OFF;
  float* lsum = reinterpret_cast<float*>(smem + F_LSUM_OFF);  // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + F_BAR_OFF);
  uint64_t* q_full = bars;                 // [kQB]
  uint64_t* q_empty = q_full + kQB;        // [kQB]
  uint64_t* k_full = q_empty + kQB;        // [kKS]
  uint64_t* k_empty = k_full + kKS;        // [kKS]
  uint64_t* v_full = k_empty + kKS;        // [kVS]
  uint64_t* v_empty = v_full + kVS;        // [kVS]
  uint64_t* s_full = v_empty + kVS;        // [2] per slot
  uint64_t* p_full = s_full + 2;           // [2]
  uint64_t* o_full = p_full + 2;           // [2]
  uint64_t* o_empty = o_full + 2;          // [2]
  uint64_t* l_full = o_empty + 2;          // [2]
  uint64_t* l_empty = l_full + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(l_empty + 2);

  const int n_pairs = (n_tiles + 1) / 2;
  const int n_work = n_pairs * n_heads;
  const int d = n_heads * kFHD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* const fa_trace = g_fa_trace;
  if (threadIdx.x == 0) FA_TRACE(224);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    for (int i = 0; i < kQB; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    for (int i = 0; i < kKS; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < kVS; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_full[x], 1);
      mbar_init(&p_full[x], 128);
      mbar_init(&o_full[x], 1);
      mbar_init(&o_empty[x], 128);
      mbar_init(&l_full[x], 128);
      mbar_init(&l_empty[x], 128);
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

  // registers: producers / MMA 80, softmax 2 x 184, epilogue 64 (x 128 threads = 64K)
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 80;" ::: "memory");
    if (lane == 0 && (warp == 0 || warp == 3)) {
      // --------------------------------------------------- K / V producers
      const bool is_k = warp == 0;
      const uint64_t keep = policy_evict_last();  // prefix K/V: re-read by every tile
      const int col0 = (is_k ? d : 2 * d);
      uint8_t* ring = is_k ? sK : sV;
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      const int stages = is_k ? kKS : kVS;
      int L = 0;
      FaWork w;
      for (int item = blockIdx.x; item < n_work; item += gridDim.x) {
        w.load(tiles, n_tiles, n_pairs, item);
        for (int i = 0; i < w.rounds; ++i) {
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            if (i >= w.s[x].n || (x == 1 && i < w.nsh)) continue;
            int kb, ke;
            w.s[x].block(i, kb, ke);
            const int st = L % stages;
            mbar_wait(&empty[st], ((L / stages) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[st], kFTile);
            for (int b = 0; b < 2; ++b)
              tma_load_2d_hint(&tm_qkv, &full[st], ring + st * kFTile + b * kFBox,
                               col0 + w.h * kFHD + b * 64, kb, keep);
            ++L;
          }
        }
      }
    } else if (lane == 0 && warp == 2) {
      // ------------------------------------------------------ Q producer
      int qi = 0;
      FaWork w;
      for (int item = blockIdx.x; item < n_work; item += gridDim.x) {
        w.load(tiles, n_tiles, n_pairs, item);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          if (x == 1 && !w.two) break;
          const int qb = qi % kQB;
          mbar_wait(&q_empty[qb], ((qi / kQB) & 1) ^ 1);
          mbar_arrive_expect_tx(&q_full[qb], kFTile);
          for (int b = 0; b < 2; ++b)
            tma_load_2d(&tm_qkv, &q_full[qb], sQ + qb * kFTile + b * kFBox,
                        w.h * kFHD + b * 64, w.s[x].t.q_begin);
          ++qi;
        }
      }
    } else if (lane == 0 && warp == 1) {
      // ------------------------------------------------------------- MMA
      constexpr uint32_t idesc_pv = idesc_bf16_f32_bmn(kFTM, kFHD);
      struct Pend {
        bool on, first, last, rel;
        int load, nk;
      } pend[2] = {{false, false, false, false, 0, 0}, {false, false, false, false, 0, 0}};
      int pcnt[2] = {0, 0};   // PVs issued per slot (p_full phase)
      int ocnt[2] = {0, 0};   // tiles finished per slot (o_empty phase)
      int qbuf[2] = {0, 0}, qph[2] = {0, 0};
      int L = 0, qi = 0, ev = 0;
      auto do_pv = [&](int x) __attribute__((always_inline)) {
        Pend& p = pend[x];
        if (p.first) mbar_wait(&o_empty[x], (ocnt[x] & 1) ^ 1);
        if (ev < 16) FA_TRACE(6 * ev + 0);
        mbar_wait(&p_full[x], pcnt[x] & 1);
        if (ev < 16) FA_TRACE(6 * ev + 1);
        ++pcnt[x];
        mbar_wait(&v_full[p.load % kVS], (p.load / kVS) & 1);
        if (ev < 16) FA_TRACE(6 * ev + 2);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sV + (p.load % kVS) * kFTile);
        for (int s = 0; s < p.nk; ++s)
          umma_bf16_ts(tmem + F_O_COL + x * 128, tmem + F_S_COL + x * 128 + s * 8,
                       sw128_mnmajor_desc(v_addr + s * 16 * 128, kFBox, 1024), idesc_pv,
                       (!p.first || s > 0) ? 1u : 0u);
        if (ev < 16) FA_TRACE(6 * ev + 3);
        if (p.rel) umma_commit(&v_empty[p.load % kVS]);
        if (p.last) {
          umma_commit(&o_full[x]);
          ++ocnt[x];
        }
        p.on = false;
      };
      FaWork w;
      for (int item = blockIdx.x; item < n_work; item += gridDim.x) {
        w.load(tiles, n_tiles, n_pairs, item);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          if (x == 1 && !w.two) break;
          qbuf[x] = qi % kQB;
          qph[x] = (qi / kQB) & 1;
          ++qi;
        }
        for (int i = 0; i < w.rounds; ++i) {
          int ld0 = 0;
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            if (pend[x].on) do_pv(x);
            if (i >= w.s[x].n) continue;
            const bool shared = i < w.nsh;
            const int ld = (x == 1 && shared) ? ld0 : L++;
            if (x == 0) ld0 = ld;
            int kb, ke;
            w.s[x].block(i, kb, ke);
            const int nkeys = (ke - kb + 31) & ~31;
            if (i == 0) mbar_wait(&q_full[qbuf[x]], qph[x]);
            mbar_wait(&k_full[ld % kKS], (ld / kKS) & 1);
            if (ev < 16) FA_TRACE(6 * ev + 4);
            tc_fence_after();
            const uint32_t q_addr = smem_u32(sQ + qbuf[x] * kFTile);
            const uint32_t k_addr = smem_u32(sK + (ld % kKS) * kFTile);
            const uint32_t idesc_s = idesc_bf16_f32(kFTM, nkeys);
#pragma unroll
            for (int s = 0; s < kFHD / 16; ++s) {
              const uint32_t off = (s >> 2) * kFBox + (s & 3) * 32;
              umma_bf16(tmem + F_S_COL + x * 128, sw128_kmajor_desc(q_addr + off),
                        sw128_kmajor_desc(k_addr + off), idesc_s, s > 0 ? 1u : 0u);
            }
            const bool rel = !(shared && x == 0 && w.s[1].n > i);
            if (rel) umma_commit(&k_empty[ld % kKS]);
            if (i == w.s[x].n - 1) umma_commit(&q_empty[qbuf[x]]);
            umma_commit(&s_full[x]);
            if (ev < 16) FA_TRACE(6 * ev + 5);
            ++ev;
            pend[x] = {true, i == 0, i == w.s[x].n - 1, rel, ld, nkeys / 16};
          }
        }
      }
#pragma unroll
      for (int x = 0; x < 2; ++x)
        if (pend[x].on) do_pv(x);
    }
    __syncwarp();
  } else if (warp < 12) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 184;" ::: "memory");
    // ---------------------------------------------------------- softmax
    const int x = (warp - 4) >> 2;      // slot
    const int quad = warp & 3;          // TMEM lane quadrant
    const int r = quad * 32 + lane;     // tile row of this thread
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t s_col = tmem + lane_off + F_S_COL + x * 128;
    const uint32_t o_col = tmem + lane_off + F_O_COL + x * 128;
    const float scale_log2 = 1.4426950408889634f * rsqrtf(static_cast<float>(kFHD));
    int sc = 0, ic = 0;
    FaWork w;
    for (int item = blockIdx.x; item < n_work; item += gridDim.x) {
      w.load(tiles, n_tiles, n_pairs, item);
      if (x == 1 && !w.two) continue;
      FaTile T;  // this slot's tile, in registers (w.s[x] with a runtime x lives in local memory)
      T.set(x == 0 ? tiles[2 * (item - w.h * n_pairs)] : tiles[2 * (item - w.h * n_pairs) + 1]);
      const int row = T.t.q_begin + r;
      const bool live = row < T.t.q_end;
      RowSpan sp = {0, 0, 0, 0};
      if (live) sp = spans[row];
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < T.n; ++j) {
        int kb, ke;
        T.block(j, kb, ke);
        const int nch = (ke - kb + 31) >> 5;
        mbar_wait(&s_full[x], sc & 1);
        if (quad == 0 && lane == 0 && sc < 20) FA_TRACE(96 + 48 * x + 2 * sc);
        ++sc;
        tc_fence_after();
        uint32_t s[kFBK];  // raw fp32 bits of S, masked in place
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c < nch) tmem_ld_32x32b_x32(s_col + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[c * 32]));
        constexpr uint32_t kNegInf = 0xff800000u;
        // visibility (independent of S: computed while the TMEM load is in flight)
        // key visible iff in [kb, ke) and in ([pb, pe) U [ss, row])
        const int a_lo = max(kb, sp.prefix_begin) - kb, a_hi = min(ke, sp.prefix_end) - kb;
        const int b_lo = max(kb, sp.span_start) - kb, b_hi = min(ke, row + 1) - kb;
        const bool full = live && ke - kb == kFBK &&
                          ((a_lo <= 0 && a_hi >= kFBK) || (b_lo <= 0 && b_hi >= kFBK));
        const bool all_full = __all_sync(0xffffffffu, full);
        uint32_t mk[4];
#pragma unroll
        for (int c = 0; c < 4; ++c)
          mk[c] = all_full ? 0xffffffffu
                           : (live && c < nch ? (fa_bits(a_lo, a_hi, c) | fa_bits(b_lo, b_hi, c)) : 0u);
        tmem_ld_wait();
        bool chunk_on[4];
        if (all_full) {
#pragma unroll
          for (int c = 0; c < 4; ++c) chunk_on[c] = true;
        } else {
          // branch-free masking (per-chunk branches around the register
          // array made ptxas spill); chunks no row of the warp sees skip the
          // exponentials below
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            chunk_on[c] = __any_sync(0xffffffffu, mk[c] != 0u);
#pragma unroll
            for (int i = 0; i < 32; ++i) s[c * 32 + i] = ((mk[c] >> i) & 1u) ? s[c * 32 + i] : kNegInf;
          }
        }
        float mx;
        {
          float m8[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) m8[c] = fmaxf(__uint_as_float(s[2 * c]), __uint_as_float(s[2 * c + 1]));
#pragma unroll
          for (int i = 16; i < kFBK; i += 16)
#pragma unroll
            for (int c = 0; c < 8; ++c)
              m8[c] = fmax3f(m8[c], __uint_as_float(s[i + 2 * c]), __uint_as_float(s[i + 2 * c + 1]));
          mx = fmaxf(fmax3f(m8[0], m8[1], m8[2]),
                     fmax3f(fmaxf(m8[3], m8[4]), fmax3f(m8[5], m8[6], m8[7]), -INFINITY));
        }
        const bool move =
            mx > m_used && (m_used == -INFINITY || (mx - m_used) * scale_log2 > kFRescaleLog2);
        const float m_new = move ? mx : m_used;
        if (j > 0 && __any_sync(0xffffffffu, move)) {
          // Every PV of this tile so far used the old base (S_j complete =>
          // PV_{j-1} complete: one thread issues both, in order).
          const float corr = move ? ex2_approx((m_used - m_new) * scale_log2) : 1.f;
          l *= corr;
#pragma unroll 1
          for (int cc = 0; cc < kFHD / 32; ++cc) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(o_col + cc * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
            tmem_st_32x32b_x32(o_col + cc * 32, v);
          }
        }
        m_used = m_new;
        const float base = m_used == -INFINITY ? 0.f : m_used * scale_log2;
        const uint64_t sc2 = f32x2(scale_log2, scale_log2), nb2 = f32x2(-base, -base);
        uint64_t acc0 = f32x2(0.f, 0.f), acc1 = acc0;
        // P chunk c (16 bf16x2 columns) goes over S columns [16c, 16c + 16),
        // whose S values are already in registers.
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c >= nch) break;
          uint32_t pk[16];
          if (chunk_on[c]) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const uint64_t a2 = fma_f32x2(f32x2(__uint_as_float(s[c * 32 + i]),
                                                  __uint_as_float(s[c * 32 + i + 1])), sc2, nb2);
              float p0, p1;
              if (kFPoly > 0 && (i >> 1) % kFPoly == kFPoly - 1) {
                f32x2_split(ex2_poly_x2(a2), p0, p1);  // this pair on the FMA pipe
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
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = 0u;
          }
          tmem_st_32x32b_x16(s_col + c * 16, pk);
        }
        float r0, r1, r2, r3;
        f32x2_split(acc0, r0, r1);
        f32x2_split(acc1, r2, r3);
        l += (r0 + r1) + (r2 + r3);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[x]);
        if (quad == 0 && lane == 0 && sc <= 20) FA_TRACE(96 + 48 * x + 2 * (sc - 1) + 1);
      }
      // row sum -> epilogue warpgroup
      mbar_wait(&l_empty[x], (ic & 1) ^ 1);
      lsum[x * 128 + r] = l;
      mbar_arrive(&l_full[x]);
      ++ic;
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;" ::: "memory");
    // --------------------------------------------------------- epilogue
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    int ec[2] = {0, 0};
    FaWork w;
    for (int item = blockIdx.x; item < n_work; item += gridDim.x) {
      w.load(tiles, n_tiles, n_pairs, item);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        if (x == 1 && !w.two) break;
        const int row = w.s[x].t.q_begin + r;
        const bool live = row < w.s[x].t.q_end;
        const uint32_t ph = ec[x] & 1;
        mbar_wait(&l_full[x], ph);
        const int te = ec[0] + ec[1];
        if (quad == 0 && lane == 0 && te < 8) FA_TRACE(192 + 4 * te);
        const float lv = lsum[x * 128 + r];
        mbar_arrive(&l_empty[x]);
        mbar_wait(&o_full[x], ph);
        if (quad == 0 && lane == 0 && te < 8) FA_TRACE(192 + 4 * te + 1);
        tc_fence_after();
        const float inv = lv > 0.f ? 1.f / lv : 0.f;
        __nv_bfloat16* dst = out + static_cast<size_t>(row) * d + w.h * kFHD;
#pragma unroll 1
        for (int cc = 0; cc < kFHD / 32; ++cc) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(tmem + lane_off + F_O_COL + x * 128 + cc * 32, v);
          tmem_ld_wait();
          if (live) {
            uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float* f = reinterpret_cast<const float*>(&v[q * 8]);
              d4[q] = make_uint4(pack_bf16x2(f[0] * inv, f[1] * inv), pack_bf16x2(f[2] * inv, f[3] * inv),
                                 pack_bf16x2(f[4] * inv, f[5] * inv), pack_bf16x2(f[6] * inv, f[7] * inv));
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&o_empty[x]);
        if (quad == 0 && lane == 0 && te < 8) FA_TRACE(192 + 4 * te + 2);
        ++ec[x];
      }
    }
  }

  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
  if (threadIdx.x == 0) FA_TRACE(225);
}

}  // namespace

cudaError_t attention_fa_set_trace(unsigned long long* dev_buf) {
  return cudaMemcpyToSymbol(g_fa_trace, &dev_buf, sizeof(dev_buf));
}

// Opt-in (SRK_ATTN=fa); measured slower than the single-tile kernel at C2
// (DESIGN.md §4, 2.05 vs 1.52 ms of attention per query).
bool attn_use_fa() {
  static const bool fa = [] {
    const char* v = std::getenv("SRK_ATTN");
    return v != nullptr && v[0] == 'f';
  }();
  return fa;
}

cudaError_t attention_fa(const CUtensorMap& tm_qkv, const RowSpan* spans, const AttnTile* tiles,
                         int n_tiles, __nv_bfloat16* out, int n_heads, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(attn_fa_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  const int work = (n_tiles + 1) / 2 * n_heads;
  const int grid = work < num_sms(dev) ? work : num_sms(dev);
  return launch_k(attn_fa_kernel, dim3(grid), dim3(kFThreads), F_SMEM, stream, tm_qkv, spans,
                  tiles, n_tiles, out, n_heads);
}

}  // namespace srk
