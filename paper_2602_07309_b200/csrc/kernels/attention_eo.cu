// Segment-masked shared-prefix attention with de-phased softmax warps (head 128).
//
// Same semantics as kernels/attention_tc.cu (reference kernels.cpp:51-95 with
// the multi-item mask of engine.cpp:147-184): query row r attends keys
// [prefix_begin, prefix_end) U [span_start, r]; softmax(q.k / sqrt(hd)) V.
//
// Why: the single-tile kernel's phase trace (tools/attn_phases.py) shows a
// 128-key block costs ~2.45k cycles per SM sub-partition, of which the
// exponentials are ~1.45k (MUFU-bound: 2 warps x 64 keys x 32 rows) and the
// TMEM load / mask / max / pair exchange / P store ~0.9k — serial, because the
// two softmax warps of a sub-partition split the keys of the same block and
// meet at the max exchange every block, so MUFU idles while both load and
// reduce. Here the two warps of a sub-partition own alternate BLOCKS instead
// (global block parity): each handles all 128 keys of its blocks with its own
// running max / sum and its own O accumulator in TMEM, so one warp's load /
// max phase overlaps the other's exponentials, and no exchange is needed.
// The epilogue merges the two partial softmaxes per row:
//   O = (O0 2^(m0 - m) + O1 2^(m1 - m)) / (l0 2^(m0 - m) + l1 2^(m1 - m)).
//
// Persistent: one CTA per SM walks (128-row tile, head) work items; the block
// sequence is continuous across items (attn_blocks.cuh schedule).
//   warp 0 TMA K, warp 3 TMA V (2-stage rings), warp 2 TMA Q (2 buffers by
//   item parity), warp 1 TMEM alloc + single-thread tcgen05.mma issuer:
//     S_g = Q K_g^T -> S[g & 1];  O[g & 1] += P_g V_g (P over S[g & 1])
//   warps 4-7  softmax of even blocks, warps 8-11 odd blocks (one thread per
//              row, lazy rescale of its own O), warps 12-15 epilogue.
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).
#include <cuda_bf16.h>

#include <cstdlib>

#include "attn_blocks.cuh"
#include "launch.h"
#include "ptx.cuh"

namespace srk {

namespace {

using attn::FaTile;
using attn::fa_bits;
using attn::kFBK;

constexpr int kEHD = 128;
constexpr int kETM = 128;
constexpr int kEBox = 16384;
constexpr int kETile = 2 * kEBox;
constexpr int kEThreads = 512;
constexpr float kERescaleLog2 = 8.0f;

constexpr int E_Q_OFF = 0;                     // 2 buffers (item parity)
constexpr int E_K_OFF = E_Q_OFF + 2 * kETile;  // 2 stages
constexpr int E_V_OFF = E_K_OFF + 2 * kETile;  // 2 stages
constexpr int E_ML_OFF = E_V_OFF + 2 * kETile;  // [2 slots][2 (m, l)][128]
constexpr int E_BAR_OFF = E_ML_OFF + 2 * 2 * 128 * 4;
constexpr int E_SMEM = E_BAR_OFF + 256 + 1024;
static_assert(E_SMEM <= 232448, "attention_eo: shared memory budget");
constexpr uint32_t E_S_COL = 0, E_O_COL = 256;

// Optional per-CTA clock64 timeline (tuning only, attention_set_trace):
// softmax slot x own block k < 24: 2 (24 x + k) + {0 S seen, 1 P handed};
// MMA block g < 32: 96 + 2 g + {0 PV waits done, 1 next S issued}; 224 / 225
// start / end.
__device__ unsigned long long* g_eo_trace = nullptr;
#define EO_TRACE(slot)                                                                     \
  do {                                                                                     \
    if (eo_trace != nullptr && (slot) < 256)                                               \
      eo_trace[blockIdx.x * 256 + (slot)] = static_cast<unsigned long long>(clock64());    \
  } while (0)

// Walks the (item, block) sequence of one CTA.
struct EoCursor {
  int li = -1;  // local item counter
  int item = 0, h = 0, j = 0;
  FaTile T;
  bool valid = false;
  __device__ void next_item(const AttnTile* tiles, int n_tiles, int n_items, int item_) {
    do {
      ++li;
      item = item_;
      valid = item < n_items;
      if (!valid) return;
      h = item / n_tiles;
      T.set(tiles[item - h * n_tiles]);
      j = 0;
      item_ += gridDim.x;
    } while (T.n == 0);
  }
  // advance one block; true when a new item started
  __device__ bool advance(const AttnTile* tiles, int n_tiles, int n_items) {
    if (++j < T.n) return false;
    next_item(tiles, n_tiles, n_items, item + gridDim.x);
    return true;
  }
};

__global__ void __launch_bounds__(kEThreads, 1)
    attn_eo_kernel(const __grid_constant__ CUtensorMap tm_qkv, const RowSpan* __restrict__ spans,
                   const AttnTile* __restrict__ tiles, int n_tiles, __nv_bfloat16* __restrict__ out,
                   int n_heads) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + E_Q_OFF;
  uint8_t* sK = smem + E_K_OFF;
  uint8_t* sV = smem + E_V_OFF;
  float* ml = reinterpret_cast<float*>(smem + E_ML_OFF);  // [x][0 = m, 1 = l][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + E_BAR_OFF);
  uint64_t* q_full = bars + 0;    // [2] item parity
  uint64_t* q_empty = bars + 2;   // [2]
  uint64_t* k_full = bars + 4;    // [2] block parity
  uint64_t* k_empty = bars + 6;
  uint64_t* v_full = bars + 8;
  uint64_t* v_empty = bars + 10;
  uint64_t* s_full = bars + 12;   // [2] slot (= block parity)
  uint64_t* p_full = bars + 14;   // [2]
  uint64_t* o_empty = bars + 16;  // [2] per O buffer
  uint64_t* l_full = bars + 18;   // [2] per slot
  uint64_t* l_empty = bars + 20;  // [2]
  uint64_t* o_full = bars + 22;   // [1] the item's last PV is done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 23);

  const int n_items = n_tiles * n_heads;
  const int d = n_heads * kEHD;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* const eo_trace = g_eo_trace;
  if (threadIdx.x == 0) EO_TRACE(224);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_empty[i], 128);
      mbar_init(&l_full[i], 128);
      mbar_init(&l_empty[i], 128);
    }
    mbar_init(o_full, 1);
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

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 64;" ::: "memory");
    if (lane == 0 && (warp == 0 || warp == 3)) {
      // --------------------------------------------------- K / V producers
      const bool is_k = warp == 0;
      const uint64_t keep = policy_evict_last();  // prefix K/V: re-read by every tile
      const int col0 = is_k ? d : 2 * d;
      uint8_t* ring = is_k ? sK : sV;
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      EoCursor c;
      c.next_item(tiles, n_tiles, n_items, blockIdx.x);
      for (int g = 0; c.valid; ++g) {
        int kb, ke;
        c.T.block(c.j, kb, ke);
        const int st = g & 1;
        mbar_wait(&empty[st], ((g >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[st], kETile);
        for (int b = 0; b < 2; ++b)
          tma_load_2d_hint(&tm_qkv, &full[st], ring + st * kETile + b * kEBox,
                           col0 + c.h * kEHD + b * 64, kb, keep);
        c.advance(tiles, n_tiles, n_items);
      }
    } else if (lane == 0 && warp == 2) {
      // ------------------------------------------------------ Q producer
      EoCursor c;
      c.next_item(tiles, n_tiles, n_items, blockIdx.x);
      while (c.valid) {
        const int qb = c.li & 1;
        mbar_wait(&q_empty[qb], ((c.li >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], kETile);
        for (int b = 0; b < 2; ++b)
          tma_load_2d(&tm_qkv, &q_full[qb], sQ + qb * kETile + b * kEBox, c.h * kEHD + b * 64,
                      c.T.t.q_begin);
        c.j = c.T.n - 1;
        c.advance(tiles, n_tiles, n_items);
      }
    } else if (lane == 0 && warp == 1) {
      // ------------------------------------------------------------- MMA
      constexpr uint32_t idesc_pv = idesc_bf16_f32_bmn(kETM, kEHD);
      EoCursor sc, pc;  // next block to issue S for / PV for
      sc.next_item(tiles, n_tiles, n_items, blockIdx.x);
      pc = sc;
      int gs = 0;
      auto issue_s = [&]() {
        const int qb = sc.li & 1;
        if (sc.j == 0) mbar_wait(&q_full[qb], (sc.li >> 1) & 1);
        int kb, ke;
        sc.T.block(sc.j, kb, ke);
        const uint32_t idesc_s = idesc_bf16_f32(kETM, (ke - kb + 31) & ~31);
        mbar_wait(&k_full[gs & 1], (gs >> 1) & 1);
        tc_fence_after();
        const uint32_t q_addr = smem_u32(sQ + qb * kETile);
        const uint32_t k_addr = smem_u32(sK + (gs & 1) * kETile);
#pragma unroll
        for (int s = 0; s < kEHD / 16; ++s) {
          const uint32_t off = (s >> 2) * kEBox + (s & 3) * 32;
          umma_bf16(tmem + E_S_COL + (gs & 1) * 128, sw128_kmajor_desc(q_addr + off),
                    sw128_kmajor_desc(k_addr + off), idesc_s, s > 0 ? 1u : 0u);
        }
        umma_commit(&k_empty[gs & 1]);
        if (sc.j == sc.T.n - 1) umma_commit(&q_empty[qb]);  // the item's last S
        umma_commit(&s_full[gs & 1]);
        ++gs;
        sc.advance(tiles, n_tiles, n_items);
      };
      if (sc.valid) issue_s();
      if (sc.valid) issue_s();
      // first block of each parity in the current PV item (accumulate = 0)
      bool fresh[2] = {true, true};
      for (int g = 0; pc.valid; ++g) {
        const int x = g & 1;
        if (pc.j == 0) fresh[0] = fresh[1] = true;
        if (fresh[x]) mbar_wait(&o_empty[x], (pc.li & 1) ^ 1);  // epilogue drained O[x]
        mbar_wait(&p_full[x], (g >> 1) & 1);
        mbar_wait(&v_full[x], (g >> 1) & 1);
        if (g < 32) EO_TRACE(96 + 2 * g);
        tc_fence_after();
        int kb, ke;
        pc.T.block(pc.j, kb, ke);
        const int nk = ((ke - kb + 31) & ~31) / 16;
        const uint32_t v_addr = smem_u32(sV + x * kETile);
        for (int s = 0; s < nk; ++s)
          umma_bf16_ts(tmem + E_O_COL + x * 128, tmem + E_S_COL + x * 128 + s * 8,
                       sw128_mnmajor_desc(v_addr + s * 16 * 128, kEBox, 1024), idesc_pv,
                       (!fresh[x] || s > 0) ? 1u : 0u);
        fresh[x] = false;
        umma_commit(&v_empty[x]);
        if (pc.j == pc.T.n - 1) umma_commit(o_full);  // every PV of the item is done
        // S_{g+2} reuses S[x], whose P_g the PV just issued reads (in order)
        if (sc.valid) issue_s();
        if (g < 32) EO_TRACE(97 + 2 * g);
        pc.advance(tiles, n_tiles, n_items);
      }
    }
    __syncwarp();
  } else if (warp < 12) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 184;" ::: "memory");
    // ---------------------------------------------------------- softmax
    const int x = (warp - 4) >> 2;      // block parity this warpgroup owns
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t s_col = tmem + lane_off + E_S_COL + x * 128;
    const uint32_t o_col = tmem + lane_off + E_O_COL + x * 128;
    const float scale_log2 = 1.4426950408889634f * rsqrtf(static_cast<float>(kEHD));
    EoCursor c;
    c.next_item(tiles, n_tiles, n_items, blockIdx.x);
    int g = 0, sc = 0;
    while (c.valid) {
      const int li = c.li;
      const int row = c.T.t.q_begin + r;
      const bool live = row < c.T.t.q_end;
      RowSpan sp = {0, 0, 0, 0};
      if (live) sp = spans[row];
      float m_used = -INFINITY, l = 0.f;
      bool mine_before = false;  // this warp already owns a block of this item
      bool item_done = false;
      while (!item_done) {
        if ((g & 1) == x) {
          int kb, ke;
          c.T.block(c.j, kb, ke);
          const int nch = (ke - kb + 31) >> 5;
          mbar_wait(&s_full[x], sc & 1);
          if (quad == 0 && lane == 0 && sc < 24) EO_TRACE(2 * (24 * x + sc));
          ++sc;
          tc_fence_after();
          uint32_t s[kFBK];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            if (cc < nch)
              tmem_ld_32x32b_x32(s_col + cc * 32, *reinterpret_cast<uint32_t(*)[32]>(&s[cc * 32]));
          constexpr uint32_t kNegInf = 0xff800000u;
          const int a_lo = max(kb, sp.prefix_begin) - kb, a_hi = min(ke, sp.prefix_end) - kb;
          const int b_lo = max(kb, sp.span_start) - kb, b_hi = min(ke, row + 1) - kb;
          const bool full = live && ke - kb == kFBK &&
                            ((a_lo <= 0 && a_hi >= kFBK) || (b_lo <= 0 && b_hi >= kFBK));
          const bool all_full = __all_sync(0xffffffffu, full);
          uint32_t mk[4];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc)
            mk[cc] = all_full ? 0xffffffffu
                              : (live && cc < nch ? (fa_bits(a_lo, a_hi, cc) | fa_bits(b_lo, b_hi, cc))
                                                  : 0u);
          tmem_ld_wait();
          bool chunk_on[4];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            chunk_on[cc] = all_full || __any_sync(0xffffffffu, mk[cc] != 0u);
            if (!all_full) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                s[cc * 32 + i] = ((mk[cc] >> i) & 1u) ? s[cc * 32 + i] : kNegInf;
            }
          }
          float mx;
          {
            float m8[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
              m8[q] = fmaxf(__uint_as_float(s[2 * q]), __uint_as_float(s[2 * q + 1]));
#pragma unroll
            for (int i = 16; i < kFBK; i += 16)
#pragma unroll
              for (int q = 0; q < 8; ++q)
                m8[q] = fmax3f(m8[q], __uint_as_float(s[i + 2 * q]), __uint_as_float(s[i + 2 * q + 1]));
            mx = fmaxf(fmax3f(m8[0], m8[1], m8[2]),
                       fmax3f(fmaxf(m8[3], m8[4]), fmax3f(m8[5], m8[6], m8[7]), -INFINITY));
          }
          const bool move =
              mx > m_used && (m_used == -INFINITY || (mx - m_used) * scale_log2 > kERescaleLog2);
          const float m_new = move ? mx : m_used;
          if (mine_before && __any_sync(0xffffffffu, move)) {
            // this warp's earlier PVs of the item used the old base (S_g
            // complete => PV_{g-2} complete: issued before it by one thread)
            const float corr = move ? ex2_approx((m_used - m_new) * scale_log2) : 1.f;
            l *= corr;
#pragma unroll 1
            for (int cc = 0; cc < kEHD / 32; ++cc) {
              uint32_t v[32];
              tmem_ld_32x32b_x32(o_col + cc * 32, v);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * corr);
              tmem_st_32x32b_x32(o_col + cc * 32, v);
            }
          }
          m_used = m_new;
          mine_before = true;
          const float base = m_used == -INFINITY ? 0.f : m_used * scale_log2;
          const uint64_t sc2 = f32x2(scale_log2, scale_log2), nb2 = f32x2(-base, -base);
          uint64_t acc0 = f32x2(0.f, 0.f), acc1 = acc0;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            if (cc >= nch) break;
            uint32_t pk[16];
            if (chunk_on[cc]) {
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                const uint64_t a2 = fma_f32x2(f32x2(__uint_as_float(s[cc * 32 + i]),
                                                    __uint_as_float(s[cc * 32 + i + 1])), sc2, nb2);
                float a0, a1;
                f32x2_split(a2, a0, a1);
                const float p0 = ex2_approx(a0), p1 = ex2_approx(a1);
                if (i & 2) acc1 = add_f32x2(acc1, f32x2(p0, p1));
                else acc0 = add_f32x2(acc0, f32x2(p0, p1));
                pk[i >> 1] = pack_bf16x2(p0, p1);
              }
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) pk[i] = 0u;
            }
            tmem_st_32x32b_x16(s_col + cc * 16, pk);
          }
          float r0, r1, r2, r3;
          f32x2_split(acc0, r0, r1);
          f32x2_split(acc1, r2, r3);
          l += (r0 + r1) + (r2 + r3);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&p_full[x]);
          if (quad == 0 && lane == 0 && sc <= 24) EO_TRACE(2 * (24 * x + sc - 1) + 1);
        }
        ++g;
        item_done = c.advance(tiles, n_tiles, n_items);
      }
      // this warp's (m, l) of the item -> epilogue (m = -inf, l = 0 if it owned no block)
      mbar_wait(&l_empty[x], (li & 1) ^ 1);
      ml[(x * 2 + 0) * 128 + r] = m_used;
      ml[(x * 2 + 1) * 128 + r] = l;
      mbar_arrive(&l_full[x]);
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 80;" ::: "memory");
    // --------------------------------------------------------- epilogue
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const float scale_log2 = 1.4426950408889634f * rsqrtf(static_cast<float>(kEHD));
    EoCursor c;
    c.next_item(tiles, n_tiles, n_items, blockIdx.x);
    int g0 = 0;  // global index of the item's first block
    while (c.valid) {
      const int li = c.li, h = c.h;
      const int row = c.T.t.q_begin + r;
      const bool live = row < c.T.t.q_end;
      // which O buffers hold this item's blocks (parity of its blocks)
      const bool has0 = c.T.n >= 2 || (g0 & 1) == 0;
      const bool has1 = c.T.n >= 2 || (g0 & 1) == 1;
      mbar_wait(&l_full[0], li & 1);
      mbar_wait(&l_full[1], li & 1);
      const float m0 = ml[0 * 128 + r], l0 = ml[1 * 128 + r];
      const float m1 = ml[2 * 128 + r], l1 = ml[3 * 128 + r];
      mbar_arrive(&l_empty[0]);
      mbar_arrive(&l_empty[1]);
      const float mm = fmaxf(m0, m1);
      const float a0 = m0 == -INFINITY ? 0.f : ex2_approx((m0 - mm) * scale_log2);
      const float a1 = m1 == -INFINITY ? 0.f : ex2_approx((m1 - mm) * scale_log2);
      const float L = l0 * a0 + l1 * a1;
      const float inv = L > 0.f ? 1.f / L : 0.f;
      const float c0 = a0 * inv, c1 = a1 * inv;
      mbar_wait(o_full, li & 1);
      tc_fence_after();
      __nv_bfloat16* dst = out + static_cast<size_t>(row) * d + h * kEHD;
#pragma unroll 1
      for (int cc = 0; cc < kEHD / 32; ++cc) {
        uint32_t v0[32], v1[32];
        if (has0) tmem_ld_32x32b_x32(tmem + lane_off + E_O_COL + cc * 32, v0);
        if (has1) tmem_ld_32x32b_x32(tmem + lane_off + E_O_COL + 128 + cc * 32, v1);
        tmem_ld_wait();
        float f[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float o0 = has0 ? __uint_as_float(v0[i]) * c0 : 0.f;
          f[i] = has1 ? fmaf(__uint_as_float(v1[i]), c1, o0) : o0;
        }
        if (live) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + cc * 32);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            d4[q] = make_uint4(pack_bf16x2(f[8 * q], f[8 * q + 1]), pack_bf16x2(f[8 * q + 2], f[8 * q + 3]),
                               pack_bf16x2(f[8 * q + 4], f[8 * q + 5]),
                               pack_bf16x2(f[8 * q + 6], f[8 * q + 7]));
        }
      }
      tc_fence_before();
      mbar_arrive(&o_empty[0]);
      mbar_arrive(&o_empty[1]);
      g0 += c.T.n;
      c.j = c.T.n - 1;
      c.advance(tiles, n_tiles, n_items);
    }
  }

  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, 512);
  if (threadIdx.x == 0) EO_TRACE(225);
}

}  // namespace

cudaError_t attention_eo_set_trace(unsigned long long* dev_buf) {
  return cudaMemcpyToSymbol(g_eo_trace, &dev_buf, sizeof(dev_buf));
}

// Opt-in until measured (SRK_ATTN=eo).
bool attn_use_eo() {
  static const bool eo = [] {
    const char* v = std::getenv("SRK_ATTN");
    return v != nullptr && v[0] == 'e';
  }();
  return eo;
}

cudaError_t attention_eo(const CUtensorMap& tm_qkv, const RowSpan* spans, const AttnTile* tiles,
                         int n_tiles, __nv_bfloat16* out, int n_heads, cudaStream_t stream) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(attn_eo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, E_SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  const int work = n_tiles * n_heads;
  const int grid = work < num_sms(dev) ? work : num_sms(dev);
  return launch_k(attn_eo_kernel, dim3(grid), dim3(kEThreads), E_SMEM, stream, tm_qkv, spans,
                  tiles, n_tiles, out, n_heads);
}

}  // namespace srk
