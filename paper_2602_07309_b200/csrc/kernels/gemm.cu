// Host launchers for the tcgen05 GEMM (gemm_tcgen05.cuh).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gemm_tcgen05.cuh"
#include "launch.h"

namespace srk {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
  });
  return fn;
}

// Output map for the epilogue's TMA store / add-reduce: [M x N] with row
// pitch ldo, 32-row x 128-byte boxes, 128 B swizzle (matches the staging
// layout written by the epilogue warps). Rows >= M are clipped by TMA.
template <int EPI>
cudaError_t make_out_map(CUtensorMap* map, void* out, int M, int N, int ldo) {
  auto fn = get_encode_fn();
  if (fn == nullptr) return cudaErrorNotSupported;
  constexpr bool f32 = EpiOut<EPI>::F32;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(M)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldo) * (f32 ? 4 : 2)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(EpiOut<EPI>::CW), 32};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int BN, int EPI>
cudaError_t launch_one(const CUtensorMap& tmA, const CUtensorMap& tmB, int M, int N, int K,
                       void* out, int ldo, cudaStream_t stream) {
  using C = GemmCfg<BN>;
  auto kern = gemm_bf16_tcgen05_kernel<BN, EPI>;
  static bool attr_set = false;  // benign race: idempotent attribute set
  if (!attr_set) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  const int tiles = ((M + C::BM - 1) / C::BM) * (N / BN);
  const int grid = tiles < num_sms(dev) ? tiles : num_sms(dev);
  if (grid <= 0) return cudaSuccess;
  CUtensorMap tmC;
  cudaError_t e = make_out_map<EPI>(&tmC, out, M, N, ldo);
  if (e != cudaSuccess) return e;
  return launch_k(kern, dim3(grid), dim3(C::THREADS), C::SMEM_BYTES, stream, tmA, tmB, tmC, M, N, K);
}

template <int BN>
cudaError_t launch_bn(const CUtensorMap& tmA, const CUtensorMap& tmB, int M, int N, int K,
                      void* out, int ldo, int epi, cudaStream_t stream) {
  switch (epi) {
    case EPI_BF16: return launch_one<BN, EPI_BF16>(tmA, tmB, M, N, K, out, ldo, stream);
    case EPI_GELU_BF16: return launch_one<BN, EPI_GELU_BF16>(tmA, tmB, M, N, K, out, ldo, stream);
    case EPI_RESID_F32: return launch_one<BN, EPI_RESID_F32>(tmA, tmB, M, N, K, out, ldo, stream);
    case EPI_F32: return launch_one<BN, EPI_F32>(tmA, tmB, M, N, K, out, ldo, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// Pairs per cluster: 1 by default. SRK_GEMM_NP=2 selects the 4-CTA cluster
// with A multicast (N % 512 == 0). Measured on B200 (C2 shapes): per-tile
// main-loop time is identical with and without the multicast (the loop is not
// L2-bandwidth bound at 6 stages), so the 16 SMs a 4-CTA grid leaves idle
// make it slower; kept for tuning on other shapes / parts.
int gemm_pairs_per_cluster(int N) {
  static const int forced = [] {
    const char* v = std::getenv("SRK_GEMM_NP");
    return v != nullptr ? std::atoi(v) : 0;
  }();
  if (N % (2 * GemmPairCfg<EPI_BF16>::BN) == 0 && forced == 2) return 2;
  return 1;
}

template <int EPI, int NP>
cudaError_t launch_pair(const CUtensorMap& tmA, const CUtensorMap& tmB, int M, int N, int K,
                        void* out, int ldo, const GemmLnArgs& ln, int rev, cudaStream_t stream) {
  using C = GemmPairCfg<EPI>;
  auto kern = gemm_bf16_tcgen05_pair_kernel<EPI, NP>;
  static int max_clusters = 0;  // co-resident clusters of 2*NP CTAs (per process, one GPU type)
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2 * NP;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.blockDim = dim3(C::THREADS, 1, 1);
  cfg.dynamicSmemBytes = C::SMEM_BYTES;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (max_clusters == 0) {
    cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cfg.gridDim = dim3(2 * NP * (num_sms(dev) / (2 * NP)), 1, 1);
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    if (e != cudaSuccess) return e;
    if (n <= 0) return cudaErrorInvalidConfiguration;
    max_clusters = n;
  }
  const int tiles = ((M + 2 * C::BM - 1) / (2 * C::BM)) * (N / (NP * C::BN));
  const int clusters = tiles < max_clusters ? tiles : max_clusters;
  if (clusters <= 0) return cudaSuccess;
  CUtensorMap tmC;
  cudaError_t e = make_out_map<EPI>(&tmC, out, M, N, ldo);
  if (e != cudaSuccess) return e;
  cfg.gridDim = dim3(2 * NP * clusters, 1, 1);
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  e = cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmC, ln, M, N, K, rev);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int EPI>
cudaError_t launch_pair_np(const CUtensorMap& tmA, const CUtensorMap& tmB, int M, int N, int K,
                           void* out, int ldo, const GemmLnArgs& ln, int rev, cudaStream_t stream) {
  if (gemm_pairs_per_cluster(N) == 2)
    return launch_pair<EPI, 2>(tmA, tmB, M, N, K, out, ldo, ln, rev, stream);
  return launch_pair<EPI, 1>(tmA, tmB, M, N, K, out, ldo, ln, rev, stream);
}

cudaError_t gemm_bf16_pair(const CUtensorMap& tmA, const CUtensorMap& tmB, int M, int N, int K,
                           void* out, int ldo, int epi, cudaStream_t stream, const LnFold* fold,
                           bool rev) {
  if (M <= 0) return cudaSuccess;
  if (N % GemmPairCfg<EPI_BF16>::BN != 0 || K % 8 != 0) return cudaErrorInvalidValue;
  GemmLnArgs ln;
  std::memset(&ln, 0, sizeof(ln));
  ln.resid_out = static_cast<float*>(out);
  ln.resid_ld = ldo;
  if (epi == EPI_RESID_LN) {
    if (fold == nullptr || fold->xb == nullptr || fold->stats_out == nullptr || fold->ld < M)
      return cudaErrorInvalidValue;
    cudaError_t e = make_out_map<EPI_BF16>(&ln.tm_xb, fold->xb, M, N, ldo);
    if (e != cudaSuccess) return e;
    ln.stats_out = reinterpret_cast<float2*>(fold->stats_out);
    ln.ld = fold->ld;
  } else if (epi == EPI_RESID_F32_LN) {
    if (fold == nullptr || fold->ln_cnt == nullptr) return cudaErrorInvalidValue;
    ln.ln_cnt = fold->ln_cnt;
  } else if (epi == EPI_LN_BF16 || epi == EPI_LN_GELU_BF16) {
    if (fold == nullptr || fold->stats_in == nullptr || fold->colsum == nullptr ||
        fold->n_parts < 1 || fold->n_parts > 16 || K % fold->n_parts != 0 || fold->ld < M)
      return cudaErrorInvalidValue;
    ln.stats_in = reinterpret_cast<const float2*>(fold->stats_in);
    ln.colsum = fold->colsum;
    ln.n_parts = fold->n_parts;
    ln.ld = fold->ld;
  }
  switch (epi) {
    case EPI_BF16: return launch_pair_np<EPI_BF16>(tmA, tmB, M, N, K, out, ldo, ln, rev ? 1 : 0, stream);
    case EPI_GELU_BF16:
      return launch_pair_np<EPI_GELU_BF16>(tmA, tmB, M, N, K, out, ldo, ln, rev ? 1 : 0, stream);
    case EPI_RESID_F32:
      return launch_pair_np<EPI_RESID_F32>(tmA, tmB, M, N, K, out, ldo, ln, rev ? 1 : 0, stream);
    case EPI_F32: return launch_pair_np<EPI_F32>(tmA, tmB, M, N, K, out, ldo, ln, rev ? 1 : 0, stream);
    case EPI_RESID_LN:
      return launch_pair_np<EPI_RESID_LN>(tmA, tmB, M, N, K, out, ldo, ln, rev ? 1 : 0, stream);
    case EPI_RESID_F32_LN:
      return launch_pair_np<EPI_RESID_F32_LN>(tmA, tmB, M, N, K, out, ldo, ln, rev ? 1 : 0, stream);
    case EPI_LN_BF16: return launch_pair_np<EPI_LN_BF16>(tmA, tmB, M, N, K, out, ldo, ln, rev ? 1 : 0, stream);
    case EPI_LN_GELU_BF16:
      return launch_pair_np<EPI_LN_GELU_BF16>(tmA, tmB, M, N, K, out, ldo, ln, rev ? 1 : 0, stream);
  }
  return cudaErrorInvalidValue;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("SRK_PDL");
    return v == nullptr || std::atoi(v) != 0;
  }();
  return on;
}

int num_sms(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (cached[device] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    cached[device] = n > 0 ? n : 148;
  }
  return cached[device];
}

cudaError_t make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                              uint32_t box_rows, uint32_t box_cols) {
  auto fn = get_encode_fn();
  if (fn == nullptr) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

int gemm_pick_bn(int N) {
  if (N % 256 == 0) return 256;
  if (N % 128 == 0) return 128;
  if (N % 64 == 0) return 64;
  return 0;
}

cudaError_t gemm_bf16(const CUtensorMap& tmA, const CUtensorMap& tmB, int M, int N, int K,
                      void* out, int ldo, int epi, int bn, cudaStream_t stream) {
  if (M <= 0) return cudaSuccess;
  if (N % bn != 0 || K % 8 != 0) return cudaErrorInvalidValue;
  switch (bn) {
    case 256: return launch_bn<256>(tmA, tmB, M, N, K, out, ldo, epi, stream);
    case 128: return launch_bn<128>(tmA, tmB, M, N, K, out, ldo, epi, stream);
    case 64: return launch_bn<64>(tmA, tmB, M, N, K, out, ldo, epi, stream);
  }
  return cudaErrorInvalidValue;
}

cudaError_t gemm_set_trace(unsigned long long* dev_buf) {
  return cudaMemcpyToSymbol(g_gemm_trace, &dev_buf, sizeof(dev_buf));
}

}  // namespace srk
