// Host-side launch interface for the sm_100a kernels (internal; the public
// boundary is include/semrank_b200.h).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <utility>
#include <vector>

namespace srk {

// Programmatic dependent launch for the forward's kernels (SRK_PDL=0 turns it
// off): a kernel may be scheduled while its predecessor drains, and must pass
// pdl_wait() before touching anything the predecessor wrote (or still reads);
// pdl_trigger() lets its own successor launch; every kernel triggers once its
// own work is done (successors then overlap only the teardown + launch).
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
#endif
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Row descriptor for segment-masked attention (one per packed row).
// Row r may attend keys [prefix_begin, prefix_end) U [span_start, r]
// (kernels.hpp:39-46 MaskSpan, generalised with prefix_begin so several
// queries can share one packed batch).
struct RowSpan {
  int32_t prefix_begin;
  int32_t prefix_end;
  int32_t span_start;
  int32_t pad;
};

// One attention work tile: query rows [q_begin, q_end) and the two key ranges
// that cover every key any of those rows may see.
struct AttnTile {
  int32_t q_begin, q_end;
  int32_t r1_begin, r1_end;  // shared-prefix keys
  int32_t r2_begin, r2_end;  // own-segment keys
  int32_t pad0, pad1;
};

// ------------------------------------------------------------------- GEMM
// Fused epilogues (gemm_tcgen05.cuh):
//   EPI_BF16      Q|K|V projection -> bf16 (model.cpp:189-196)
//   EPI_GELU_BF16 W_in + exact-erf GELU -> bf16 (model.cpp:206-209, kernels.cpp:47-49)
//   EPI_RESID_F32 x += acc, fp32 residual stream (model.cpp:199-202, 210-213)
//   EPI_F32       plain fp32 store (tests)
//   EPI_RESID_LN / EPI_LN_BF16 / EPI_LN_GELU_BF16: LayerNorm folded into the
//                 projections (pair kernel only, see LnFold below)
enum GemmEpilogue : int {
  EPI_BF16 = 0, EPI_GELU_BF16 = 1, EPI_RESID_F32 = 2, EPI_F32 = 3,
  EPI_RESID_LN = 4, EPI_LN_BF16 = 5, EPI_LN_GELU_BF16 = 6, EPI_RESID_F32_LN = 7
};
int num_sms(int device);
cudaError_t make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                              uint32_t box_rows, uint32_t box_cols);
// Picks BN from N; N must be a multiple of 64, K a multiple of 8.
int gemm_pick_bn(int N);
cudaError_t gemm_bf16(const CUtensorMap& tmA, const CUtensorMap& tmB, int M, int N, int K,
                      void* out, int ldo, int epi, int bn, cudaStream_t stream);
// LayerNorm folded into the projections (gemm_tcgen05.cuh, GemmLnArgs).
// epi 4 (residual + LN statistics): out = x fp32 [M x N] += acc, xb = bf16(x),
//   stats_out[N/128][ld] = per-row (mean, M2) float2 partials over 128 columns.
// epi 5 / 6 (normalised projection [+ GELU]): A = xb, B = diag(gain) W (bf16),
//   out = bf16([gelu](rstd * (acc - mean * colsum))), mean/rstd from
//   stats_in[n_parts][ld] (each part over K / n_parts columns).
// epi 7 (residual with completion counts): out = x fp32 += acc as epi 2, and
//   ln_cnt[r / 128] += 1 once a CTA's add-reductions into 128-row block r are
//   complete (N / 256 per block); layer_norm_after() waits on them.
struct LnFold {
  unsigned int* ln_cnt = nullptr;
  __nv_bfloat16* xb = nullptr;
  float* stats_out = nullptr;       // float2 pairs
  const float* stats_in = nullptr;  // float2 pairs
  const float* colsum = nullptr;
  int n_parts = 0;
  int ld = 0;
};
// CTA-pair (cta_group::2) 256 x 256 tiles; N % 256 == 0; tmA and tmB both use
// 128-row x 64-column boxes. Epilogues 4-6 need `fold`.
cudaError_t gemm_bf16_pair(const CUtensorMap& tmA, const CUtensorMap& tmB, int M, int N, int K,
                           void* out, int ldo, int epi, cudaStream_t stream,
                           const LnFold* fold = nullptr, bool rev = false);
// The projection GEMMs take the pair path when N is a multiple of 256.
inline bool gemm_use_pair(int N) { return N % 256 == 0; }
// B-operand box rows for a weight [N x K] map on the chosen path.
inline int gemm_b_box_rows(int N) { return gemm_use_pair(N) ? 128 : gemm_pick_bn(N); }
// Dispatch: pair kernel when N % 256 == 0, else the 1-CTA kernel.
inline cudaError_t gemm_auto(const CUtensorMap& tmA, const CUtensorMap& tmB, int M, int N, int K,
                             void* out, int ldo, int epi, cudaStream_t stream,
                             const LnFold* fold = nullptr, bool rev = false) {
  // rev: 256-row blocks in reverse order (L2 serpentine; pair kernel only)
  if (gemm_use_pair(N)) return gemm_bf16_pair(tmA, tmB, M, N, K, out, ldo, epi, stream, fold, rev);
  if (epi > 3) return cudaErrorInvalidValue;  // LN folding is a pair-kernel epilogue
  return gemm_bf16(tmA, tmB, M, N, K, out, ldo, epi, gemm_pick_bn(N), stream);
}

// ------------------------------------------------------------ elementwise
// x[r] = (src[r] >= 0 ? tok_emb[src[r]] : soft[-src[r]-1]) + pos_emb[pos[r]]
// and xn[r] = bf16(LN(x[r]) * gain) (layer-0 LN1 fused).
cudaError_t embed_ln(const int32_t* src, const int32_t* pos, const float* tok_emb,
                     const float* soft_rows, const float* pos_emb, const float* gain, float* x,
                     __nv_bfloat16* xn, int M, int d, cudaStream_t stream);
// Folded-LN path: x as above, xb = bf16(x), stats[0][row] = (mean, M2) of x.
cudaError_t embed_stats(const int32_t* src, const int32_t* pos, const float* tok_emb,
                        const float* soft_rows, const float* pos_emb, float* x,
                        __nv_bfloat16* xb, float* stats, int M, int d, cudaStream_t stream);
// Mixed-mode items given as compact embeddings [n x d_emb]:
// zero-pad form (service.cpp:208-217): out [n x d] = emb[:, :min(d_emb, d)], 0 after;
// projection operand: out [n x kp] bf16, columns >= d_emb zero.
cudaError_t emb_pad_rows(const float* emb, int n, int d_emb, int d, float* out,
                         cudaStream_t stream);
cudaError_t emb_to_bf16(const float* emb, int n, int d_emb, int kp, __nv_bfloat16* out,
                        cudaStream_t stream);
// LayerNorm that runs concurrently with a residual GEMM (epi 7, another
// stream): 128-row block b is normalised once cnt[b] == contrib, then cnt[b]
// is reset to 0 for the next GEMM. Needs the GEMM co-resident (it is: this
// kernel uses no shared memory and one 256-thread CTA per SM).
cudaError_t layer_norm_after(const float* x, const float* gain, __nv_bfloat16* out, int M, int d,
                             unsigned int* cnt, int contrib, cudaStream_t stream);
// rev: rows walked from the last block to the first (L2 serpentine order).
cudaError_t layer_norm_bf16(const float* x, const float* gain, __nv_bfloat16* out, int M, int d,
                            cudaStream_t stream, bool rev = false);

// -------------------------------------------------------------- attention
// qkv: [M x 3d] bf16 rows (q | k | v); out: [M x d] bf16.
cudaError_t attention(const __nv_bfloat16* qkv, const RowSpan* spans, const AttnTile* tiles,
                      int n_tiles, __nv_bfloat16* out, int M, int n_heads, int head_dim,
                      cudaStream_t stream);
// tcgen05/TMEM path for head_dim in {64, 128}; tm_qkv maps the [rows x 3d]
// bf16 qkv buffer with 64 x 128 boxes (make_tmap_bf16_2d(.., 128, 64)).
// work / n_work: optional device work list from attention_work_lpt (item ->
// (tile, head)); nullptr = head-major order.
cudaError_t attention_tc(const CUtensorMap& tm_qkv, const void* qkv, const RowSpan* spans,
                         const AttnTile* tiles, int n_tiles, __nv_bfloat16* out, int M,
                         int n_heads, int head_dim, cudaStream_t stream,
                         const int2* work = nullptr, int n_work = 0);
// Longest-processing-time assignment of the (tile, head) work items to the
// persistent attention CTAs (cost = key blocks of the tile + per-item
// overhead), laid out for the kernel's strided walk: out[k * ctas + c] is the
// k-th item of CTA c, (-1, 0) where a CTA has fewer. ctas = attention_ctas().
int attention_ctas(int n_tiles, int n_heads, int device);
void attention_work_lpt(const AttnTile* tiles, int n_tiles, int n_heads, int ctas,
                        std::vector<int2>& out);
// Tuning aid: per-CTA clock64 timeline of attention_tc (nullptr disables).
cudaError_t attention_set_trace(unsigned long long* dev_buf);
cudaError_t gemm_set_trace(unsigned long long* dev_buf);
// Query rows per attention tile for a head size (128 on the tcgen05 path).
int attention_tile_rows(int head_dim);

// -------------------------------------------------------- score head/topk
// Final LN on the last-token rows + task-column dot products + probabilities.
// w_cols: [C x d] fp32 (columns of the score head), bias: [C].
// col_kind/arity describe how columns map to tasks (see engine.cu).
cudaError_t score_head(const float* x, const int32_t* last_rows, int n_items, int d,
                       const float* ln_gain, const float* w_cols, const float* bias, int n_cols,
                       const int32_t* task_col, const int32_t* task_arity, int n_tasks,
                       int yes_col, int no_col, double* scores, float* hidden_out,
                       cudaStream_t stream);

// Service post-processing of the raw scores [n x stride] (service.cpp:242-277):
// calibrated relevance (isotonic blocks, interleaved lo/hi/value) and the
// optional task blend; out[n] is the key the page top-k sorts by.
cudaError_t final_scores(const double* scores, int stride, int n, const double* blocks,
                         int n_blocks, const int32_t* blend_task, const double* blend_w,
                         int n_blend, double* out, cudaStream_t stream);

// Base64 (base64.cpp:60-108) of n_items payloads: text [char_begin[i],
// char_end[i]) (lengths multiples of 4) -> bytes at out + byte_off[i] (out
// may be null: validate only). first_err (preset to ~0) receives
// min(item-ordered position << 2 | kind), kind 1 misplaced padding, 2 invalid
// character; positions grow with the item index (the host orders spans so).
cudaError_t b64_decode(const uint8_t* text, const int64_t* char_begin, const int64_t* char_end,
                       const int64_t* byte_off, int n_items, uint8_t* out,
                       unsigned long long* first_err, cudaStream_t stream);

struct TopkEntry {
  double score;
  int64_t id;
  int32_t index;
  int32_t pad;
};
// Per segment s (items [seg_off[s], seg_off[s+1])): the k best entries by
// (score desc, id asc, index asc). scores has stride `stride`.
// max_seg_len bounds the longest segment (sizes the chunking).
cudaError_t topk(const double* scores, int stride, const int64_t* ids, const int32_t* seg_off,
                 int n_segments, int max_seg_len, int k, TopkEntry* scratch, int scratch_cap,
                 TopkEntry* out, cudaStream_t stream);
// Merge: entries [n] (already candidates) -> best k.
cudaError_t topk_merge(const TopkEntry* in, int n, int k, TopkEntry* out, cudaStream_t stream);
// Best k of any number of entries (multi-level: groups of 4096 -> k each);
// k <= kTopkSelectMaxK; scratch holds topk_select_scratch(n, k) entries.
constexpr int kTopkSelectMaxK = 2048;
size_t topk_select_scratch(long long n, int k);
cudaError_t topk_select(const TopkEntry* in, long long n, int k, TopkEntry* scratch,
                        TopkEntry* out, cudaStream_t stream);

// ------------------------------------------------- exhaustive retrieval scan
// Reference: exhaustive_topk (retrieval.cpp:134-173) with rar_score
// (:60-71) = w0 * cosine(q, e_d) (double accumulation, :44-58) + sum w_i f_i.
// Pass 1 (HBM-bound): fp32 scores with a rigorous error bound eps; each CTA
// keeps every doc within 2 eps of its running k-th best (a superset of its
// exact top-k). Pass 2: the candidates are rescored in double in the
// reference's operation order. Pass 3: exact top-k (score desc, id asc).
struct RetrievalScan {
  const float* emb;       // [n x D]
  const float* feat;      // [n x F] (may be null when F == 0)
  const int64_t* ids;     // [n]
  const uint8_t* keep;    // [n] filter mask or null
  const float* q32;       // [D]
  const double* qd;       // [D] (query as double)
  const float* w32;       // [F]
  const double* wd;       // [F]
  double w0;
  double q_norm;          // sqrt(sum double(q_i)^2), the reference's sqrt(na)
  float eps2;             // 2 * fp32 error bound of a score
  long long n;
  int D, F, k;
};
// cand: int32 [cand_cap]; counters: int32 [2] = {count, flags} (zeroed by the
// call); flags bit 0 = a kept doc has a zero embedding, bit 1 = candidate
// overflow (the exact fallback path must run).
cudaError_t retrieval_scan(const RetrievalScan& a, int32_t* cand, int cand_cap, int32_t* counters,
                           int grid, cudaStream_t stream);
// Large k (> 512): full stable sort of n entries by (score desc, id asc)
// (device radix sorts), first min(k, n) gathered to out.
size_t retrieval_sort_scratch(long long n);
cudaError_t retrieval_sort_topk(const TopkEntry* e, long long n, int k, void* scratch,
                                size_t scratch_bytes, TopkEntry* out, cudaStream_t stream);
// Exact double rescoring of cand[0..n_cand) (or of all docs when cand is null
// and n_cand == n) into entries.
cudaError_t retrieval_refine(const RetrievalScan& a, const int32_t* cand, long long n_cand,
                             TopkEntry* out, int32_t* counters, cudaStream_t stream);

// ------------------------------------------------------------ conversions
// dst[n][k] = bf16(src[k][n]) : fp32 [K x N] row-major -> bf16 [N x K].
// scale_k (device, optional): dst[n][k] = bf16(src[k][n] * scale_k[k]) (LN gain folding).
cudaError_t transpose_to_bf16(const float* src, __nv_bfloat16* dst, int K, int N,
                              cudaStream_t stream, const float* scale_k = nullptr);
// out[n] = sum_k float(w[n][k]) for bf16 w [N x K] (folded-LN column sums).
cudaError_t bf16_row_sums(const __nv_bfloat16* w, int N, int K, float* out, cudaStream_t stream);

}  // namespace srk
