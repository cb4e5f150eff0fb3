// Key-block schedule of a 128-row query tile for the tcgen05 attention
// kernels (attention_fa.cu, attention_eo.cu): the prefix range r1 in 128-key
// blocks, then the own-segment range r2 = [r2_begin, q_end) aligned on the
// tile itself: back-aligned head blocks + the diagonal block [q_begin, q_end).
#pragma once

#include <cstdint>

#include "launch.h"

namespace srk {
namespace attn {

constexpr int kFBK = 128;  // keys per block (max)

// Bits [lo, hi) of the 32-key chunk c (key offsets relative to the block).
__device__ __forceinline__ uint32_t fa_bits(int lo, int hi, int c) {
  lo = min(max(lo - 32 * c, 0), 32);
  hi = min(max(hi - 32 * c, 0), 32);
  if (hi <= lo) return 0u;
  const uint32_t upto = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
  return upto & ~((1u << lo) - 1u);
}

// Blocks of one tile: prefix range r1 in 128-key blocks, then the own range
// r2 = [r2_begin, q_end) as back-aligned head blocks + the diagonal block.
struct FaTile {
  AttnTile t;
  int nb1 = 0, nh = 0, n = 0;
  __device__ void set(const AttnTile& tt) {
    t = tt;
    nb1 = t.r1_end > t.r1_begin ? (t.r1_end - t.r1_begin + kFBK - 1) / kFBK : 0;
    if (t.r2_end > t.r2_begin) {
      const int head = t.q_begin > t.r2_begin ? t.q_begin - t.r2_begin : 0;
      nh = (head + kFBK - 1) / kFBK;
      n = nb1 + nh + 1;
    } else {
      nh = 0;
      n = nb1;
    }
  }
  // keys [kb, ke) of block j
  __device__ void block(int j, int& kb, int& ke) const {
    if (j < nb1) {
      kb = t.r1_begin + j * kFBK;
      ke = min(kb + kFBK, t.r1_end);
      return;
    }
    const int jj = j - nb1;
    if (jj < nh) {
      kb = max(t.r2_begin, t.q_begin - kFBK * (nh - jj));
      ke = t.q_begin - kFBK * (nh - 1 - jj);
    } else {
      kb = max(t.r2_begin, t.q_begin);
      ke = t.r2_end;
    }
  }
};


}  // namespace attn
}  // namespace srk
