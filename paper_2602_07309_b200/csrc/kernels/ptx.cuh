// Inline-PTX helpers for sm_100a: mbarrier, TMA, tcgen05 (UMMA + TMEM).
//
// Encodings follow the PTX ISA for tcgen05 (shared-memory descriptor and
// instruction descriptor layouts); they were cross-checked against the CuTe
// sm100 descriptor definitions shipped in the image (flashinfer's vendored
// CUTLASS tree, cute/arch/mma_sm100_desc.hpp) but nothing is included from it.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>

namespace srk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Blocking wait for the phase with this parity. The suspend-time hint (as
// CUTLASS's ClusterBarrier) lets the hardware park the warp until the phase
// completes instead of re-polling; ncu counts ~20% of the attention kernel's
// instructions as try_wait/branch/yield, but measured per-tile and per-block
// timings are the same with and without the hint (SRK_MBAR_SUSPEND_NS=0).
#ifndef SRK_MBAR_SUSPEND_NS
#define SRK_MBAR_SUSPEND_NS 0x989680
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done;
  do {
#if SRK_MBAR_SUSPEND_NS > 0
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity), "r"(SRK_MBAR_SUSPEND_NS)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
#endif
  } while (!done);
}

// Non-blocking probe: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}

// --------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Same, with an L2 eviction-priority hint (createpolicy result).
__device__ __forceinline__ void tma_load_2d_hint(const CUtensorMap* map, uint64_t* bar, void* dst,
                                                 int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}

// smem -> global tensor tile (bulk group), and the fp32 add-reduction variant
// (the L2 performs dst += src; used for the residual-stream epilogue).
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int c0,
                                                  int c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d_hint(const CUtensorMap* map, const void* src,
                                                       int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group.L2::cache_hint"
      " [%0, {%2, %3}], [%1], %4;" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, const void* src, int c0,
                                                  int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint"
      " [%0, {%2, %3}], [%1], %4;" ::"l"(reinterpret_cast<uint64_t>(map)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
// Contiguous global bytes -> smem (1D bulk copy, completes on the mbarrier);
// 16-byte aligned addresses, size a multiple of 16.
__device__ __forceinline__ void bulk_load_1d(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Tensor tile -> L2 only (no smem destination, no completion tracking).
__device__ __forceinline__ void tma_prefetch_2d_l2(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Wait until all committed bulk groups of this thread finished reading smem.
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// Wait until at most N committed bulk groups are still reading smem.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ------------------------------------------------------------------ tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 in, fp32 accumulate, one CTA.
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]: A (M x K, K-major) lives in TMEM, one row per
// lane, two bf16 per 32-bit column (16 K-elements = 8 columns per MMA).
__device__ __forceinline__ void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive on an mbarrier once every previously issued tcgen05.mma of this
// thread has completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// Shared-memory matrix descriptor: K-major operand, 128-byte swizzle,
// 8-row core-matrix groups 1024 B apart (rows of 64 bf16 = 128 B).
//   bits  0-13 start address >> 4
//   bits 16-29 leading byte offset >> 4 (unused for swizzled K-major; 1)
//   bits 32-45 stride byte offset >> 4 (1024 B between 8-row groups)
//   bits 46-47 descriptor version (1 on sm_100)
//   bits 61-63 layout type (2 = SWIZZLE_128B)
__device__ __forceinline__ uint64_t sw128_kmajor_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// Instruction descriptor, kind::f16: bf16 A/B, fp32 D, both K-major.
//   bits 4-5 D format (1 = f32), 7-9 A format (1 = bf16), 10-12 B format,
//   15/16 A/B major (0 = K), 17-22 N >> 3, 24-28 M >> 4.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

// 32 lanes x 32 consecutive 32-bit TMEM columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
// 32 lanes x 16 consecutive 32-bit TMEM columns -> 16 registers per thread.
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// 16 lanes x 256 bits, 8 repetitions along columns (64 columns): thread t gets,
// for repetition i, lane t/4 columns 8i + 2(t%4) + {0, 1} in r[4i], r[4i+1]
// and lane t/4 + 8 in r[4i+2], r[4i+3] (CuTe SM100_TMEM_LOAD_16dp256b8x).
__device__ __forceinline__ void tmem_ld_16x256b_x8(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 registers -> 32 consecutive TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// 16 registers -> 16 consecutive TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Completed async-proxy (TMA) global writes -> ordered before this thread's
// later generic-proxy accesses (e.g. the release that publishes them).
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// 16-byte global load cached in L2 only (data another SM just wrote).
__device__ __forceinline__ float4 ld_cg_f4(const float4* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// Generic-proxy shared-memory writes -> visible to the async proxy (UMMA/TMA).
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Shared-memory matrix descriptor for an MN-major operand (N contiguous),
// 128-byte swizzle: 64-element MN chunks `lbo` bytes apart, 8-row K groups
// `sbo` bytes apart (CuTe canonical ((8,n),(8,k)):((1,LBO),(8,SBO)) in 16 B units).
__device__ __forceinline__ uint64_t sw128_mnmajor_desc(uint32_t saddr, uint32_t lbo,
                                                       uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// kind::f16 descriptor with B MN-major (bit 16) — for O += P.V with V rows
// [key][dim] used as B[k=key][n=dim].
__host__ __device__ constexpr uint32_t idesc_bf16_f32_bmn(int m, int n) {
  return idesc_bf16_f32(m, n) | (1u << 16);
}

// ------------------------------------------------------ CTA pairs (2-SM)
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Arrive on an mbarrier of another CTA of the cluster. Default (CTA-scope)
// semantics, as CUTLASS's ClusterBarrier::arrive: the payloads are ordered by
// TMA complete_tx / tcgen05 fences, and a .release.cluster arrive would emit
// a GPU-wide MEMBAR per call.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA load into this CTA's smem whose completion is signalled on the pair
// leader's mbarrier (same smem offset, peer bit cleared).
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint64_t* bar, void* dst,
                                                 int c0, int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1),
      "l"(policy)
      : "memory");
}
// Multicast variant: the box lands at the same smem offset in every CTA of
// cta_mask; each destination's completion is signalled on its pair leader's
// mbarrier.
__device__ __forceinline__ void tma_load_2d_pair_mc(const CUtensorMap* map, uint64_t* bar,
                                                    void* dst, int c0, int c1, uint16_t cta_mask,
                                                    uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5, %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1),
      "h"(cta_mask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish_pair() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}
// Pair MMA (issued by the leader CTA): M = 256 over both CTAs' smem/TMEM.
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Commit the pair's MMAs to the same mbarrier offset in both CTAs (mask 0b11).
// Arrive (when the MMAs issued so far complete) on the mbarrier at this
// offset in every CTA of cta_mask (default: the pair of cluster ranks 0/1).
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar, uint16_t cta_mask = 3) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}

// ------------------------------------------------------------- misc utils
__device__ __forceinline__ uint64_t f32x2(float lo, float hi);
__device__ __forceinline__ void f32x2_split(uint64_t v, float& lo, float& hi);
__device__ __forceinline__ uint64_t fma_f32x2(uint64_t a, uint64_t b, uint64_t c);
__device__ __forceinline__ uint64_t add_f32x2(uint64_t a, uint64_t b);
__device__ __forceinline__ uint64_t f32x2_neg(uint64_t a) { return a ^ 0x8000000080000000ull; }
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float ex2_approx(float x) {  // MUFU.EX2; ex2(-inf) = +0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA/ALU pipes (offloads MUFU, as FlashAttention-4): x = n + f
// with n = round(x) via the 1.5*2^23 magic add (no F2I, which shares the XU
// pipe with MUFU), f in [-0.5, 0.5], degree-4 Taylor polynomial for 2^f
// (rel. error < 5e-5, far below the bf16 rounding of P), exponent added as an
// integer. Inputs <= -127 flush to +0 (as ex2.approx.ftz).
__device__ __forceinline__ float ex2_poly(float x) {
  const float xc = fmaxf(x, -127.0f);
  const float t = xc + 12582912.0f;
  const float f = xc - (t - 12582912.0f);
  float p = 9.6181291076284772e-3f;
  p = fmaf(p, f, 5.5504108664821580e-2f);
  p = fmaf(p, f, 2.4022650695910071e-1f);
  p = fmaf(p, f, 6.9314718055994531e-1f);
  p = fmaf(p, f, 1.0f);
  const int e = (__float_as_int(t) - 0x4B400000) << 23;
  const float r = __int_as_float(__float_as_int(p) + e);
  return xc <= -127.0f ? 0.0f : r;
}

// Two 2^x on the FMA/ALU pipes, packed fp32x2 (FFMA2 / FADD2 for the
// reduction and the degree-4 polynomial), for the share of a softmax's
// exponentials taken off MUFU (FlashAttention-4). Same scheme as ex2_poly;
// inputs <= -126 give +0 (as ex2.approx.ftz of a masked -inf score).
#ifndef SRK_EX2_C4
#define SRK_EX2_C4 9.6181291076284772e-3f
#endif
__device__ __forceinline__ uint64_t ex2_poly_x2(uint64_t x2) {
  float x0, x1;
  f32x2_split(x2, x0, x1);
  const float c0 = fmaxf(x0, -126.0f), c1 = fmaxf(x1, -126.0f);
  const uint64_t xc = f32x2(c0, c1);
  const uint64_t magic = f32x2(12582912.0f, 12582912.0f);
  const uint64_t t = add_f32x2(xc, magic);
  const uint64_t f = add_f32x2(xc, add_f32x2(magic, f32x2_neg(t)));
  uint64_t p = fma_f32x2(f32x2(SRK_EX2_C4, SRK_EX2_C4), f,
                         f32x2(5.5504108664821580e-2f, 5.5504108664821580e-2f));
  p = fma_f32x2(p, f, f32x2(2.4022650695910071e-1f, 2.4022650695910071e-1f));
  p = fma_f32x2(p, f, f32x2(6.9314718055994531e-1f, 6.9314718055994531e-1f));
  p = fma_f32x2(p, f, f32x2(1.0f, 1.0f));
  float t0, t1, p0, p1;
  f32x2_split(t, t0, t1);
  f32x2_split(p, p0, p1);
  const float r0 = __int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23) - (0x4B400000 << 23));
  const float r1 = __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23) - (0x4B400000 << 23));
  return f32x2(c0 <= -126.0f ? 0.0f : r0, c1 <= -126.0f ? 0.0f : r1);
}

// exp2 of a packed pair on the FMA pipe, degree 3 (rel. error ~1e-4, below
// the bf16 rounding of P): x clamped to -126 so masked (-inf) inputs give
// 2^-126 (negligible next to the row max's 1) and no select is needed;
// 2^n is added to the polynomial's exponent field with one LEA per value.
__device__ __forceinline__ uint64_t ex2_poly3_x2(uint64_t x2) {
  float x0, x1;
  f32x2_split(x2, x0, x1);
  const uint64_t xc = f32x2(fmaxf(x0, -126.0f), fmaxf(x1, -126.0f));
  const uint64_t magic = f32x2(12582912.0f, 12582912.0f);
  const uint64_t t = add_f32x2(xc, magic);
  const uint64_t f = add_f32x2(xc, add_f32x2(magic, f32x2_neg(t)));
  uint64_t p = fma_f32x2(f32x2(5.5504108664821580e-2f, 5.5504108664821580e-2f), f,
                         f32x2(2.4022650695910071e-1f, 2.4022650695910071e-1f));
  p = fma_f32x2(p, f, f32x2(6.9314718055994531e-1f, 6.9314718055994531e-1f));
  p = fma_f32x2(p, f, f32x2(1.0f, 1.0f));
  float t0, t1, p0, p1;
  f32x2_split(t, t0, t1);
  f32x2_split(p, p0, p1);
  // t's low mantissa bits hold n; (t_bits << 23) == n << 23 (mod 2^32)
  return f32x2(__int_as_float(__float_as_int(p0) + (__float_as_int(t0) << 23)),
               __int_as_float(__float_as_int(p1) + (__float_as_int(t1) << 23)));
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n_threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n_threads) : "memory");
}

// Blackwell 3-input max (FMNMX3) and packed fp32x2 FMA / add (FFMA2, FADD2).
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ uint64_t f32x2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f32x2_split(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t fma_f32x2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ uint64_t add_f32x2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ float gelu_erf(float v) {
  // kernels.cpp:47-49 (reference): 0.5 v (1 + erf(v / sqrt 2)), exact erf.
  // 1 + erf(z) = 2 - erfc(z) for z >= 0 and erfc(|z|) for z < 0, with the
  // branch-free Chebyshev erfc (Numerical Recipes 6.2, fractional error
  // < 1.2e-7): two MUFU ops + 12 FMAs instead of libdevice's branchy erff,
  // and no cancellation in 1 + erf for negative v.
  const float z = fabsf(v) * 0.70710678118654752f;
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.5f, z, 1.0f)));
  float p = 0.17087277f;
  p = fmaf(p, t, -0.82215223f);
  p = fmaf(p, t, 1.48851587f);
  p = fmaf(p, t, -1.13520398f);
  p = fmaf(p, t, 0.27886807f);
  p = fmaf(p, t, -0.18628806f);
  p = fmaf(p, t, 0.09678418f);
  p = fmaf(p, t, 0.37409196f);
  p = fmaf(p, t, 1.00002368f);
  p = fmaf(p, t, -1.26551223f);
  const float erfc = t * __expf(fmaf(-z, z, p));
  const float one_plus_erf = v >= 0.0f ? 2.0f - erfc : erfc;
  return 0.5f * v * one_plus_erf;
}

__device__ __forceinline__ uint64_t mul_f32x2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// gelu_erf on a pair of values with packed fp32x2 arithmetic (FFMA2/FMUL2):
// the same Chebyshev erfc and operation order per lane as gelu_erf, half the
// FMA-pipe instructions (the W_in epilogue is issue-bound).
// SRK_GELU_AS=1 (default): Abramowitz-Stegun 7.1.26 erfc, abs. error <= 1.5e-7
// (4 packed FMAs instead of the 9 of the Numerical Recipes Chebyshev form
// below, relative error < 1.2e-7, kept as SRK_GELU_AS=0). Absolute 1.5e-7 is
// far below the bf16 rounding of the GELU output (the epilogue writes bf16);
// the W_in tile interval drops 7.17 -> 6.66 us (plain bf16 store: 6.40).
#ifndef SRK_GELU_AS
#define SRK_GELU_AS 1
#endif
__device__ __forceinline__ void gelu_erf_x2(float& v0, float& v1) {
#if SRK_GELU_AS
  // Abramowitz-Stegun 7.1.26 erfc (abs. error <= 1.5e-7): 4 FFMA2 instead of 9.
  {
    const uint64_t z = mul_f32x2(f32x2(fabsf(v0), fabsf(v1)),
                                 f32x2(0.70710678118654752f, 0.70710678118654752f));
    float z0, z1;
    f32x2_split(z, z0, z1);
#if SRK_GELU_AS == 2
    // t = 1 / (1 + p z) on the FMA pipe: z clamped to 4 (erfc(4) = 1.5e-8, the
    // clamped A-S erfc stays within 1.4e-7), d in [1, 2.31], quadratic seed
    // (rel. 3.4e-2) + two Newton steps (rel. 1.3e-6): 6 FFMA2 for 2 MUFU.RCP
    // per pair. Measured slower (W_in 1.60-1.63 vs 1.40-1.51 ms per query):
    // the W_in epilogue is FMA-issue-bound, not MUFU-bound. Off (SRK_GELU_AS=2).
    const uint64_t zc = f32x2(fminf(z0, 4.0f), fminf(z1, 4.0f));
    const uint64_t dd = fma_f32x2(f32x2(0.3275911f, 0.3275911f), zc, f32x2(1.0f, 1.0f));
    uint64_t t = fma_f32x2(fma_f32x2(f32x2(0.25461108f, 0.25461108f), dd,
                                     f32x2(-1.24656636f, -1.24656636f)),
                           dd, f32x2(1.96838612f, 1.96838612f));
    const uint64_t ndd = f32x2_neg(dd);
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const uint64_t e = fma_f32x2(ndd, t, f32x2(1.0f, 1.0f));
      t = fma_f32x2(t, e, t);
    }
#else
    float d0, d1;
    f32x2_split(fma_f32x2(f32x2(0.3275911f, 0.3275911f), z, f32x2(1.0f, 1.0f)), d0, d1);
    float t0, t1;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t0) : "f"(d0));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t1) : "f"(d1));
    const uint64_t t = f32x2(t0, t1);
#endif
    uint64_t p = fma_f32x2(f32x2(1.061405429f, 1.061405429f), t, f32x2(-1.453152027f, -1.453152027f));
    p = fma_f32x2(p, t, f32x2(1.421413741f, 1.421413741f));
    p = fma_f32x2(p, t, f32x2(-0.284496736f, -0.284496736f));
    p = fma_f32x2(p, t, f32x2(0.254829592f, 0.254829592f));
    const uint64_t arg = mul_f32x2(f32x2(-z0, -z1), mul_f32x2(z, f32x2(1.4426950408889634f, 1.4426950408889634f)));
    float a0, a1;
    f32x2_split(arg, a0, a1);
    float e0, e1;
    f32x2_split(mul_f32x2(mul_f32x2(t, p), f32x2(ex2_approx(a0), ex2_approx(a1))), e0, e1);
    const float o0 = v0 >= 0.0f ? 2.0f - e0 : e0;
    const float o1 = v1 >= 0.0f ? 2.0f - e1 : e1;
    f32x2_split(mul_f32x2(mul_f32x2(f32x2(0.5f, 0.5f), f32x2(v0, v1)), f32x2(o0, o1)), v0, v1);
    return;
  }
#endif
  const uint64_t z = mul_f32x2(f32x2(fabsf(v0), fabsf(v1)),
                               f32x2(0.70710678118654752f, 0.70710678118654752f));
  float z0, z1;
  f32x2_split(z, z0, z1);
  float d0, d1;
  f32x2_split(fma_f32x2(f32x2(0.5f, 0.5f), z, f32x2(1.0f, 1.0f)), d0, d1);
  float t0, t1;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t0) : "f"(d0));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t1) : "f"(d1));
  const uint64_t t = f32x2(t0, t1);
  uint64_t p = f32x2(0.17087277f, 0.17087277f);
  p = fma_f32x2(p, t, f32x2(-0.82215223f, -0.82215223f));
  p = fma_f32x2(p, t, f32x2(1.48851587f, 1.48851587f));
  p = fma_f32x2(p, t, f32x2(-1.13520398f, -1.13520398f));
  p = fma_f32x2(p, t, f32x2(0.27886807f, 0.27886807f));
  p = fma_f32x2(p, t, f32x2(-0.18628806f, -0.18628806f));
  p = fma_f32x2(p, t, f32x2(0.09678418f, 0.09678418f));
  p = fma_f32x2(p, t, f32x2(0.37409196f, 0.37409196f));
  p = fma_f32x2(p, t, f32x2(1.00002368f, 1.00002368f));
  p = fma_f32x2(p, t, f32x2(-1.26551223f, -1.26551223f));
  const uint64_t arg = fma_f32x2(f32x2(-z0, -z1), z, p);
  float a0, a1;
  f32x2_split(arg, a0, a1);
  float e0, e1;
  f32x2_split(mul_f32x2(t, f32x2(__expf(a0), __expf(a1))), e0, e1);
  const float o0 = v0 >= 0.0f ? 2.0f - e0 : e0;
  const float o1 = v1 >= 0.0f ? 2.0f - e1 : e1;
  f32x2_split(mul_f32x2(mul_f32x2(f32x2(0.5f, 0.5f), f32x2(v0, v1)), f32x2(o0, o1)), v0, v1);
}

}  // namespace srk
