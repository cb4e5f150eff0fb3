// Probe: cycles per tcgen05.mma (kind::f16, K = 16) for the attention kernel's
// shapes, operands resident in smem / TMEM (no TMA traffic): back-to-back
// throughput, and the time to issue 8 MMAs into an idle pipe from one thread.
// Measured on B200: ~73-84 cycles per MMA for N <= 128 (the
// 64-cycle N = 128 floor is not reached), 133 at N = 256; issuing 8 takes
// ~815 cycles (~100 per instruction) whatever N. Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//     -I paper_2602_07309_b200/csrc/kernels tools/probe/umma_rate.cu -o /tmp/umma_rate -lcuda
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace srk;

// Warp-converged issue: all 32 lanes execute, elect.sync picks the issuing lane
// inside the asm (no single-lane branch around a uniform-operand instruction).
__device__ __forceinline__ void umma_ss_e(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_ts_e(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_e(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}

__global__ void __launch_bounds__(128, 1) probe(int mode, int n, int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 196608);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 196608 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(slot, 512);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (mode >= 2 && warp == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    const uint32_t id_ss = idesc_bf16_f32(128, n);
    const uint32_t id_ts = idesc_bf16_f32_bmn(128, n);
    uint32_t ph = 0;
    long long ti = 0, tc = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      long long a0 = clock64();
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        if (mode == 2) {
          const uint32_t off = (s >> 2) * 16384 + (s & 3) * 32;
          umma_ss_e(tmem + (r & 1) * 128, sw128_kmajor_desc(a + off), sw128_kmajor_desc(b + off), id_ss, s > 0);
        } else {
          umma_ts_e(tmem + 256, tmem + s * 8, sw128_mnmajor_desc(b + s * 16 * 128, 16384, 1024), id_ts, 1);
        }
      }
      long long a1 = clock64();
      if (r < 16 || (r & 7) == 7) {
        commit_e(bar);
        mbar_wait(bar, ph);
        ph ^= 1;
      }
      long long a2 = clock64();
      if (r < 16) { ti += a1 - a0; tc += a2 - a0; }
      if (r == 15) t0 = clock64();
    }
    commit_e(bar);
    mbar_wait(bar, ph);
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      out[blockIdx.x] = static_cast<unsigned long long>((t1 - t0) * reps / (reps - 16));
      if (blockIdx.x == 0) { out[148] = ti / 16; out[149] = tc / 16; }
    }
  }
  if (mode < 2 && threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    const uint32_t id_ss = idesc_bf16_f32(128, n);
    const uint32_t id_ts = idesc_bf16_f32_bmn(128, n);
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int r = 0; r < reps; ++r) {
      if (mode == 0) {  // S = Q K^T: SS, K-major both, 8 K-steps of 16
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const uint32_t off = (s >> 2) * 16384 + (s & 3) * 32;
          umma_bf16(tmem + (r & 1) * 128, sw128_kmajor_desc(a + off), sw128_kmajor_desc(b + off),
                    id_ss, s > 0);
        }
      } else {  // O += P V: TS, A (P) from TMEM, B (V) MN-major in smem
#pragma unroll
        for (int s = 0; s < 8; ++s)
          umma_bf16_ts(tmem + 256, tmem + s * 8, sw128_mnmajor_desc(b + s * 16 * 128, 16384, 1024),
                       id_ts, 1);
      }
      if ((r & 7) == 7) {
        umma_commit(bar);
        mbar_wait(bar, ph);
        ph ^= 1;
      }
    }
    umma_commit(bar);
    mbar_wait(bar, ph);
    ph ^= 1;
    long long t1 = clock64();
    out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
    if (blockIdx.x == 0) {
      // issue latency: 8 MMAs into an idle pipe, time to issue vs time to complete
      long long ti = 0, tc = 0;
      for (int r = 0; r < 16; ++r) {
        long long a0 = clock64();
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          if (mode == 0) {
            const uint32_t off = (s >> 2) * 16384 + (s & 3) * 32;
            umma_bf16(tmem, sw128_kmajor_desc(a + off), sw128_kmajor_desc(b + off), id_ss, s > 0);
          } else {
            umma_bf16_ts(tmem + 256, tmem + s * 8, sw128_mnmajor_desc(b + s * 16 * 128, 16384, 1024),
                         id_ts, 1);
          }
        }
        long long a1 = clock64();
        umma_commit(bar);
        mbar_wait(bar, ph);
        ph ^= 1;
        long long a2 = clock64();
        ti += a1 - a0;
        tc += a2 - a0;
      }
      out[148] = ti / 16;
      out[149] = tc / 16;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 160 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[4] = {"SS (S = Q K^T)", "TS (O += P V)", "SS warp+elect", "TS warp+elect"};
  for (int mode = 0; mode < 4; ++mode)
    for (int n : {64, 128, 256}) {
      for (int grid : {1}) {
        const int reps = 4000;
        probe<<<grid, 128, 200 * 1024>>>(mode, n, reps, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        const double per = mx / (reps * 8.0);
        unsigned long long lat[2];
        cudaMemcpy(lat, d + 148, 16, cudaMemcpyDeviceToHost);
        printf("%-16s N=%3d grid %3d: %6.1f cycles per K=16 MMA (ideal %5.1f at 8192 FLOP/clk); "
               "8 MMAs into an idle pipe: issued in %llu, complete in %llu cycles %s\n",
               names[mode], n, grid, per, 128.0 * n * 16 * 2 / 8192, lat[0], lat[1],
               cudaGetErrorString(e));
      }
    }
  return 0;
}
