// Probe: MUFU exp2 throughput per SM for f32 vs packed f16x2 / bf16x2 operands
// (results per clock), 8 warps per SM, independent chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe/mufu_rate.cu -o /tmp/mufu_rate
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) v[i] = 0x3c003c00u + threadIdx.x + i;  // small positive inputs
  float f[8];
  for (int i = 0; i < 8; ++i) f[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
      if (MODE == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += f[i] + __uint_as_float(v[i]);
  if (threadIdx.x == 0) out[blockIdx.x] = (float)(t1 - t0);
  if (s == 12345.f) out[1000] = s;
}

int main() {
  float* d;
  cudaMalloc(&d, 4096 * 4);
  const int iters = 4096, threads = 256;
  const char* names[3] = {"ex2.approx.f32", "ex2.approx.f16x2", "ex2.approx.bf16x2"};
  for (int m = 0; m < 3; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) k<0><<<148, threads>>>(d, iters);
      if (m == 1) k<1><<<148, threads>>>(d, iters);
      if (m == 2) k<2><<<148, threads>>>(d, iters);
      cudaDeviceSynchronize();
    }
    float cyc;
    cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
    const double instr = (double)iters * 8 * threads;  // per SM (one CTA per SM)
    const double per_clk = instr / cyc * (m == 0 ? 1 : 2);
    printf("%-20s %.2f results/clk/SM (%.2f instr/clk) %s\n", names[m], per_clk, instr / cyc,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
