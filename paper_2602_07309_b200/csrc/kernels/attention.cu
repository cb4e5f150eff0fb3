// Segment-masked shared-prefix attention over ragged packed item segments.
//
// Reference semantics (kernels.cpp:51-95 attention_one, kernels.hpp:39-46):
// query row r, head h attends keys [prefix_begin, prefix_end) U [span_start, r],
// softmax(q.k / sqrt(hd)) with max subtraction, then the weighted V sum.
// Multi-item scoring (engine.cpp:186-236) gives every item row
// {prefix_end = T_q, span_start = item start}; prefix rows are causal.
//
// B200 design: one CTA = 64 packed query rows x one head. The host planner
// (host/planner.cpp) hands each tile two key ranges: R1 = the query's shared
// prefix (read by every item tile of that query -> L2 resident) and R2 = the
// tile's own segment keys. K/V blocks of 64 keys are staged through shared
// memory with cp.async double buffering; S = QK^T and O += PV run on bf16
// tensor cores with fp32 accumulation and an online (flash) softmax in fp32.
#include <cuda_bf16.h>

#include "launch.h"

namespace srk {

namespace {

constexpr int kBlockM = 64;
constexpr int kBlockN = 64;
constexpr int kThreads = 128;

__device__ __forceinline__ void cp_async_16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;  // src-size 0 -> zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                            uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1,
                                                  uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16_16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                               uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Shared tile [rows][HD] bf16, 16-byte chunks XOR-swizzled by row to keep
// ldmatrix conflict-free (row stride is a multiple of 128 B for HD >= 64).
template <int HD>
struct Tile {
  static constexpr int CH = HD / 8;  // 16-byte chunks per row
  static constexpr int SW = CH >= 8 ? 7 : CH - 1;
  __device__ static __forceinline__ uint32_t off(int row, int chunk) {
    return static_cast<uint32_t>((row * CH + (chunk ^ (row & SW))) * 16);
  }
};

template <int HD>
__global__ void __launch_bounds__(kThreads)
    attn_segment_kernel(const __nv_bfloat16* __restrict__ qkv, const RowSpan* __restrict__ spans,
                        const AttnTile* __restrict__ tiles, __nv_bfloat16* __restrict__ out,
                        int M, int n_heads) {
  pdl_wait();
  using T = Tile<HD>;
  constexpr int TILE_BYTES = kBlockM * HD * 2;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK = smem + TILE_BYTES;      // 2 buffers
  uint8_t* sV = smem + 3 * TILE_BYTES;  // 2 buffers
  const uint32_t sQa = static_cast<uint32_t>(__cvta_generic_to_shared(sQ));
  const uint32_t sKa = static_cast<uint32_t>(__cvta_generic_to_shared(sK));
  const uint32_t sVa = static_cast<uint32_t>(__cvta_generic_to_shared(sV));

  const AttnTile tile = tiles[blockIdx.x];
  const int h = blockIdx.y;
  const int d = n_heads * HD;
  const size_t ld = static_cast<size_t>(3) * d;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int nb1 = (tile.r1_end - tile.r1_begin + kBlockN - 1) / kBlockN;
  const int nb2 = (tile.r2_end - tile.r2_begin + kBlockN - 1) / kBlockN;
  const int nblocks = nb1 + nb2;

  // ---- Q tile -> smem
  for (int i = tid; i < kBlockM * T::CH; i += kThreads) {
    const int r = i / T::CH, c = i % T::CH;
    const int row = tile.q_begin + r;
    const bool ok = row < tile.q_end;
    const __nv_bfloat16* src = qkv + (ok ? row : 0) * ld + h * HD + c * 8;
    cp_async_16(sQa + T::off(r, c), src, ok);
  }
  auto load_kv = [&](int b, int buf) {
    int k0, kend;
    if (b < nb1) {
      k0 = tile.r1_begin + b * kBlockN;
      kend = tile.r1_end;
    } else {
      k0 = tile.r2_begin + (b - nb1) * kBlockN;
      kend = tile.r2_end;
    }
    for (int i = tid; i < kBlockN * T::CH; i += kThreads) {
      const int r = i / T::CH, c = i % T::CH;
      const int key = k0 + r;
      const bool ok = key < kend;
      const __nv_bfloat16* base = qkv + (ok ? key : 0) * ld + h * HD + c * 8;
      cp_async_16(sKa + buf * TILE_BYTES + T::off(r, c), base + d, ok);
      cp_async_16(sVa + buf * TILE_BYTES + T::off(r, c), base + 2 * d, ok);
    }
  };
  if (nblocks > 0) load_kv(0, 0);
  cp_async_commit();

  // Per-thread rows: g and g + 8 within this warp's 16-row slice.
  const int g = lane >> 2, t4 = lane & 3;
  const int row0 = tile.q_begin + warp * 16 + g;
  const int row1 = row0 + 8;
  RowSpan sp0 = {0, 0, 0, 0}, sp1 = {0, 0, 0, 0};
  if (row0 < tile.q_end) sp0 = spans[row0];
  if (row1 < tile.q_end) sp1 = spans[row1];

  const float scale_log2 = 1.4426950408889634f * rsqrtf(static_cast<float>(HD));
  float o[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  cp_async_wait<0>();
  __syncthreads();
  // Q fragments stay in registers for the whole key loop.
  uint32_t qf[HD / 16][4];
#pragma unroll
  for (int ks = 0; ks < HD / 16; ++ks) {
    const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
    const int c = ks * 2 + (lane >> 4);
    ldmatrix_x4(sQa + T::off(r, c), qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
  }

  for (int b = 0; b < nblocks; ++b) {
    const int buf = b & 1;
    if (b + 1 < nblocks) load_kv(b + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();

    int k0, kbeg, kend;
    if (b < nb1) {
      k0 = tile.r1_begin + b * kBlockN;
      kbeg = tile.r1_begin;
      kend = tile.r1_end;
    } else {
      k0 = tile.r2_begin + (b - nb1) * kBlockN;
      kbeg = tile.r2_begin;
      kend = tile.r2_end;
    }

    // S = Q K^T for this warp: 16 x 64
    float s[kBlockN / 8][4];
#pragma unroll
    for (int n = 0; n < kBlockN / 8; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
    const uint32_t kb = sKa + buf * TILE_BYTES;
#pragma unroll
    for (int ks = 0; ks < HD / 16; ++ks) {
#pragma unroll
      for (int np = 0; np < kBlockN / 16; ++np) {
        uint32_t b0, b1, b2, b3;
        const int r = np * 16 + (lane & 7) + (lane >> 4) * 8;
        const int c = ks * 2 + ((lane >> 3) & 1);
        ldmatrix_x4(kb + T::off(r, c), b0, b1, b2, b3);
        mma_bf16_16816(s[2 * np], qf[ks], b0, b1);
        mma_bf16_16816(s[2 * np + 1], qf[ks], b2, b3);
      }
    }

    // Mask + online softmax (fp32). Keys outside [kbeg, kend) belong to the
    // other range or to padding and are always excluded.
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int n = 0; n < kBlockN / 8; ++n) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int key = k0 + n * 8 + t4 * 2 + j;
        const bool inr = key >= kbeg && key < kend;
        const bool a0 = inr && ((key >= sp0.prefix_begin && key < sp0.prefix_end) ||
                                (key >= sp0.span_start && key <= row0));
        const bool a1 = inr && ((key >= sp1.prefix_begin && key < sp1.prefix_end) ||
                                (key >= sp1.span_start && key <= row1));
        s[n][j] = a0 ? s[n][j] * scale_log2 : -INFINITY;
        s[n][2 + j] = a1 ? s[n][2 + j] * scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, s[n][j]);
        mx1 = fmaxf(mx1, s[n][2 + j]);
      }
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float base0 = mn0 == -INFINITY ? 0.f : mn0;
    const float base1 = mn1 == -INFINITY ? 0.f : mn1;
    const float corr0 = exp2f(m0 - base0), corr1 = exp2f(m1 - base1);
    m0 = mn0;
    m1 = mn1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int n = 0; n < kBlockN / 8; ++n) {
      s[n][0] = exp2f(s[n][0] - base0);
      s[n][1] = exp2f(s[n][1] - base0);
      s[n][2] = exp2f(s[n][2] - base1);
      s[n][3] = exp2f(s[n][3] - base1);
      rs0 += s[n][0] + s[n][1];
      rs1 += s[n][2] + s[n][3];
    }
    l0 = l0 * corr0 + rs0;
    l1 = l1 * corr1 + rs1;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o[i][0] *= corr0;
      o[i][1] *= corr0;
      o[i][2] *= corr1;
      o[i][3] *= corr1;
    }

    // O += P V
    const uint32_t vb = sVa + buf * TILE_BYTES;
#pragma unroll
    for (int kk = 0; kk < kBlockN / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack2(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack2(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
      if constexpr (HD >= 16 && (HD / 8) % 2 == 0) {
#pragma unroll
        for (int np = 0; np < HD / 16; ++np) {
          uint32_t b0, b1, b2, b3;
          const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
          const int c = np * 2 + (lane >> 4);
          ldmatrix_x4_trans(vb + T::off(r, c), b0, b1, b2, b3);
          mma_bf16_16816(o[2 * np], pa, b0, b1);
          mma_bf16_16816(o[2 * np + 1], pa, b2, b3);
        }
      }
    }
    __syncthreads();  // buffer `buf` is overwritten by the next prefetch
  }

  // Row sums across the quad, normalise (post-normalise as the reference).
  l0 += __shfl_xor_sync(0xffffffff, l0, 1);
  l0 += __shfl_xor_sync(0xffffffff, l0, 2);
  l1 += __shfl_xor_sync(0xffffffff, l1, 1);
  l1 += __shfl_xor_sync(0xffffffff, l1, 2);
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f;
  const float inv1 = l1 > 0.f ? 1.f / l1 : 0.f;

  // Stage O through the Q tile (own 16 rows only) for coalesced 16 B stores.
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    const int c = i;  // 8-column chunk i
    const int col = t4 * 2;
    const int r0 = warp * 16 + g, r1 = r0 + 8;
    *reinterpret_cast<uint32_t*>(sQ + T::off(r0, c) + col * 2) =
        pack2(o[i][0] * inv0, o[i][1] * inv0);
    *reinterpret_cast<uint32_t*>(sQ + T::off(r1, c) + col * 2) =
        pack2(o[i][2] * inv1, o[i][3] * inv1);
  }
  __syncwarp();
  for (int i = lane; i < 16 * T::CH; i += 32) {
    const int r = warp * 16 + i / T::CH, c = i % T::CH;
    const int row = tile.q_begin + r;
    if (row < tile.q_end) {
      *reinterpret_cast<uint4*>(out + static_cast<size_t>(row) * d + h * HD + c * 8) =
          *reinterpret_cast<const uint4*>(sQ + T::off(r, c));
    }
  }
}

template <int HD>
cudaError_t launch_attn(const __nv_bfloat16* qkv, const RowSpan* spans, const AttnTile* tiles,
                        int n_tiles, __nv_bfloat16* out, int M, int n_heads,
                        cudaStream_t stream) {
  constexpr int smem = 5 * kBlockM * HD * 2;
  auto kern = attn_segment_kernel<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(n_tiles, n_heads);
  return launch_k(kern, grid, dim3(kThreads), smem, stream, qkv, spans, tiles, out, M, n_heads);
}

}  // namespace

cudaError_t attention(const __nv_bfloat16* qkv, const RowSpan* spans, const AttnTile* tiles,
                      int n_tiles, __nv_bfloat16* out, int M, int n_heads, int head_dim,
                      cudaStream_t stream) {
  if (n_tiles <= 0) return cudaSuccess;
  switch (head_dim) {
    case 16: return launch_attn<16>(qkv, spans, tiles, n_tiles, out, M, n_heads, stream);
    case 32: return launch_attn<32>(qkv, spans, tiles, n_tiles, out, M, n_heads, stream);
    case 64: return launch_attn<64>(qkv, spans, tiles, n_tiles, out, M, n_heads, stream);
    case 128: return launch_attn<128>(qkv, spans, tiles, n_tiles, out, M, n_heads, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace srk
