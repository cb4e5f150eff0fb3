// Device engine: owns bf16 K-major weights, the activation workspace, the
// packed-input buffers and captured CUDA graphs for one device/stream.
// Counterpart of ScoringEngine (engine.hpp:109-119): callers are serialised
// by a mutex exactly as ScoringEngine::score is (engine.cpp:389-392).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <vector>

#include "../kernels/launch.h"
#include "model.hpp"
#include "h2d.hpp"
#include "score_cache.hpp"
#include "planner.hpp"

namespace srh {

template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;  // elements
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
  // Returns true if (re)allocated.
  bool ensure(size_t n) {
    if (n <= cap) return false;
    release();
    size_t c = n + n / 4 + 64;
    SR_CUDA_CHECK(cudaMalloc(&ptr, c * sizeof(T)));
    cap = c;
    return true;
  }
};

template <typename T>
struct HostBuf {  // pinned
  T* ptr = nullptr;
  size_t cap = 0;
  ~HostBuf() {
    if (ptr) cudaFreeHost(ptr);
  }
  void ensure(size_t n) {
    if (n <= cap) return;
    if (ptr) cudaFreeHost(ptr);
    ptr = nullptr;
    size_t c = n + n / 4 + 64;
    SR_CUDA_CHECK(cudaMallocHost(&ptr, c * sizeof(T)));
    cap = c;
  }
};

struct LayerDev {
  __nv_bfloat16* wqkv = nullptr;  // [3d x d]
  __nv_bfloat16* wo = nullptr;    // [d x d]
  __nv_bfloat16* win = nullptr;   // [ff x d]
  __nv_bfloat16* wout = nullptr;  // [d x ff]
  float* ln1 = nullptr;
  float* ln2 = nullptr;
  // folded-LN path: wqkv / win hold diag(gain) W; their column sums
  float* cs_qkv = nullptr;  // [3d]
  float* cs_in = nullptr;   // [ff]
  CUtensorMap tm_qkv, tm_o, tm_in, tm_out;
};

class Engine;

// Kernel classes for live per-class timing (sr_plan_profile).
enum ProfClass : int {
  PROF_EMBED_LN = 0, PROF_GEMM_QKV, PROF_ATTENTION, PROF_GEMM_O, PROF_LAYERNORM, PROF_GEMM_IN,
  PROF_GEMM_OUT, PROF_SCORE_HEAD, PROF_TOPK, PROF_N
};

// Records a CUDA event pair around every launch of a profiled forward.
struct Profiler {
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
  cudaStream_t stream = nullptr;
  bool in_graph = false;  // events recorded as external nodes of a captured graph
  int cur = -1;
  cudaEvent_t cur_start = nullptr;
  void begin(int cls);
  void end();
  ~Profiler();
};

// One request shape, resident on the device, replayed through a CUDA graph.
struct Plan {
  Engine* eng = nullptr;
  PackedBatch pack;         // host copy of the packed layout
  std::vector<int32_t> layout_sig;  // layout_signature of the uploaded layout
  bool layout_ok = false;           // the device layout arrays match layout_sig
  std::vector<sr_request> reqs;
  std::vector<std::vector<int32_t>> lens;
  int32_t k = 0;
  int32_t n_tasks = 0;
  // device inputs
  DevBuf<int32_t> src, pos, last_rows, seg_off;
  DevBuf<srk::RowSpan> spans;
  DevBuf<srk::AttnTile> tiles;
  DevBuf<int2> attn_work;           // LPT order of the attention work items
  std::vector<int2> attn_work_host;
  int32_t n_attn_work = 0;
  DevBuf<int64_t> ids;
  DevBuf<float> soft;
  // outputs
  DevBuf<double> scores;
  DevBuf<double> final;  // post-processed ranking key (set_postprocess)
  DevBuf<srk::TopkEntry> topk_scratch, topk_out;
  DevBuf<srk::TopkEntry> gathered, merged;  // sharded merge
  pinned_vector<double> h_scores;           // fetch staging (page-locked)
  pinned_vector<srk::TopkEntry> h_top;
  // compact embeddings -> soft rows on the device (score_emb; -1 = none)
  int32_t emb_form = -1, emb_n = 0, emb_d = 0, emb_row0 = 0;
  std::vector<int32_t> emb_off;  // item offsets of a make_plan_emb request
  DevBuf<float> emb;
  DevBuf<__nv_bfloat16> emb16;  // projection A operand [round_up(n, 128) x kp]
  CUtensorMap tm_emb16;
  // graph
  cudaGraphExec_t graph = nullptr;
  uint64_t graph_epoch = ~0ull;  // engine workspace epoch the graph was captured at
  int32_t launches = 0;
  ~Plan();
};

class Engine {
 public:
  Engine(const ModelWeights& w, int device);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const ModelConfig& config() const { return cfg_; }
  int device() const { return device_; }
  cudaStream_t stream() const { return stream_; }
  int n_tasks() const { return 1 + static_cast<int>(cfg_.head_specs.size()); }
  std::mutex& mutex() { return mu_; }
  // LayerNorm folded into the GEMM epilogues (all projections on the pair path).
  bool fold_ln() const { return fold_ln_; }
  // Service post-processing on the device (service.cpp:242-277): calibrated
  // relevance (isotonic blocks lo/hi/value) and an optional task blend; the
  // top-k then orders by the final score. n_blocks == 0 and n_blend == 0
  // turns it off (top-k by raw relevance).
  void set_postprocess(const double* lo, const double* hi, const double* value, int n_blocks,
                       const int32_t* blend_task, const double* blend_w, int n_blend);
  bool postprocess() const { return post_on_; }
  const std::vector<double>& last_final() const { return last_final_; }

  // Builds a plan: validates + packs + uploads inputs + captures the graph.
  std::unique_ptr<Plan> make_plan(const sr_request* reqs, int n_req, int32_t k);
  // Re-uploads inputs of a same-shape request set into an existing plan.
  void refill_plan(Plan& p, const sr_request* reqs, int n_req);
  void run_plan(Plan& p);
  void fetch(Plan& p, sr_result* res, int n_req);
  // Scores + top-k through a cached plan (host buffers in, host buffers out).
  void score(const sr_request* reqs, int n_req, sr_result* res);
  void item_hidden(const sr_request& req, float* hidden_out);
  // /score wire ingest (service.cpp:326-391): mixed-mode items given as
  // base64 float32 payloads (concatenated text, char offsets [n+1]), decoded
  // on the device into the soft-row buffer (kernels/wire.cu), then scored.
  void score_b64(const int32_t* prefix, int32_t t_q, const char* text, const int64_t* char_off,
                 int32_t n_items, const int64_t* item_ids, sr_result* res);
  // Same with payload spans [begin[i], end[i]) inside text = a ++ b (the
  // JSON body and its side buffer of unescaped payloads, host/wire.hpp).
  void score_b64_spans(const int32_t* prefix, int32_t t_q, const char* a, int64_t la,
                       const char* b, int64_t lb, const int64_t* begin, const int64_t* end,
                       int32_t n_items, const int64_t* item_ids, sr_result* res);

  // Ranks given raw score rows [n x n_tasks] (host): upload, the same
  // post-processing and top-k kernels as the forward's tail, fetch. Used by
  // score_cached, whose rows come partly from the cache.
  void rank(const double* h_scores, const int64_t* ids, int32_t n, sr_result* res);
  // handle_search's cache probe (service.cpp:160-234): rows of cached items
  // come from `cache`, only the misses go through the forward (one pass, in
  // request order), their rows are put back, then all rows are ranked.
  // req.item_ids are the entity ids of the cache keys.
  void score_cached(ScoreCache& cache, const std::string& searcher_id, uint64_t signature,
                    const std::string& model_version, const sr_request& req, sr_result* res,
                    int32_t* n_hits);

  // Mixed-mode items given as compact embeddings emb [n x d_emb] (SURVEY H7,
  // north_star (d)). form SR_EMB_PAD: one soft row per item, the embedding
  // zero-padded (or cut) to d_model as the service does (service.cpp:208-217);
  // SR_EMB_PROJECT: n_soft rows per item = bf16(emb) . bf16(P) on the tensor
  // cores (fp32 accumulate), P set by set_projection. The rows are produced
  // in HBM inside the forward (no d_model-wide upload).
  void set_projection(const float* proj, int32_t d_emb, int32_t n_soft);
  void score_emb(const int32_t* prefix, int32_t t_q, const float* emb, int32_t d_emb,
                 int32_t n_items, const int64_t* item_ids, int32_t form, sr_result* res);
  std::unique_ptr<Plan> make_plan_emb(const int32_t* prefix, int32_t t_q, const float* emb,
                                      int32_t d_emb, int32_t n_items, const int64_t* item_ids,
                                      int32_t form, int32_t k);

  // Sharded: local pass + NCCL all-gather of per-rank top-k + merge.
  void run_plan_sharded(Plan& p, struct Comm* comm);

  // Enqueue the full forward for the plan's packed batch on stream_.
  int32_t enqueue_forward(Plan& p, float* hidden_out, Profiler* prof = nullptr);
  // Graph replay of the forward with an event pair around every launch;
  // per-class mean ms and launch counts per forward, averaged over `reps`.
  void profile(Plan& p, int reps, float* ms_out, int32_t* launches_out);

  // sr_engine_reserve: workspace for passes of up to M packed rows
  void reserve(int32_t M) {
    SR_CUDA_CHECK(cudaSetDevice(device_));
    ensure_workspace(M);
  }

 private:
  void ensure_workspace(int32_t M);

  ModelConfig cfg_;
  int device_;
  cudaStream_t stream_ = nullptr;
  std::mutex mu_;
  // weights
  float* tok_emb_ = nullptr;
  float* pos_emb_ = nullptr;
  float* ln_f_ = nullptr;
  float* head_w_ = nullptr;   // [C x d]
  float* head_b_ = nullptr;   // [C]
  int32_t* task_col_ = nullptr;
  int32_t* task_arity_ = nullptr;
  int n_cols_ = 0, yes_col_ = 0, no_col_ = 0;
  bool fold_ln_ = false;
  bool serpentine_ = false;
  // LayerNorm finished by the residual GEMMs' last contributor per 128-row
  // block (EPI_RESID_F32_LN) instead of separate LayerNorm launches.
  bool ln_after_ = false;
  bool attn_lpt_ = true;
  bool layout_reuse_ = true;
  std::vector<int32_t> sig_;  // layout_signature scratch
  cudaStream_t side_ = nullptr;  // LN-after kernels (concurrent with the residual GEMM)
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  bool post_on_ = false;
  int post_nblocks_ = 0, post_nblend_ = 0;
  DevBuf<double> post_blocks_, post_w_;
  DevBuf<int32_t> post_task_;
  std::vector<double> last_final_;
  // rank(): device rows, ids, one segment, top-k
  DevBuf<double> rk_scores_, rk_final_;
  DevBuf<int64_t> rk_ids_;
  DevBuf<int32_t> rk_seg_;
  DevBuf<srk::TopkEntry> rk_scratch_, rk_out_;
  // pending base64 source of the mixed request being packed (score_b64)
  struct B64Src {
    const char* a = nullptr;  // text = a ++ b
    int64_t la = 0;
    const char* b = nullptr;
    int64_t lb = 0;
    std::vector<int64_t> spans;  // begin[n] ++ end[n] ++ byte_off[n]
    int32_t n = 0;
  } b64_;
  DevBuf<uint8_t> b64_text_;
  DevBuf<int64_t> b64_off_;
  DevBuf<unsigned long long> b64_err_;
  void upload_b64_text();
  // pending compact-embedding source of the request being packed (score_emb)
  struct EmbSrc {
    const float* emb = nullptr;
    int32_t n = 0, d_emb = 0, form = -1;
  } emb_;
  std::vector<int32_t> emb_request(const int32_t* prefix, int32_t t_q, const float* emb,
                                   int32_t d_emb, int32_t n_items, const int64_t* item_ids,
                                   int32_t form, sr_request* req);
  // projection P as the UMMA B operand: bf16 [n_soft*d x proj_kp_] (K-major,
  // K zero-padded to a multiple of 64)
  DevBuf<__nv_bfloat16> proj_;
  CUtensorMap tm_proj_;
  int32_t proj_demb_ = 0, proj_kp_ = 0, proj_nsoft_ = 0;
  StagedUpload up_;  // caller-buffer uploads (soft rows, base64 text)
  std::vector<LayerDev> layers_;
  std::vector<void*> allocs_;
  // workspace
  int32_t ws_rows_ = 0;
  DevBuf<float> x_;
  DevBuf<__nv_bfloat16> xn_, qkv_, h_;
  DevBuf<__nv_bfloat16> xb_;   // folded LN: bf16 copy of the residual stream (GEMM A operand)
  DevBuf<unsigned int> ln_cnt_;  // LN-after: add-reductions per 128-row block (mod d / 256)
  DevBuf<float> stats_;        // folded LN: [d/128][ws_rows_] (mean, M2) partials
  CUtensorMap tm_xn_, tm_h_, tm_qkv_, tm_xb_;
  uint64_t ws_epoch_ = 0;  // bumps when workspace moves (graphs must be re-captured)
  // shape-keyed plan cache for score()
  std::map<std::tuple<int32_t, int32_t, int32_t, int32_t, int32_t, int32_t, int32_t, int32_t>,
           std::unique_ptr<Plan>>
      cache_;
  void capture(Plan& p);
 public:
  uint64_t epoch() const { return ws_epoch_; }
};

// ---------------------------------------------------------------- NCCL
struct Comm {
  void* nccl = nullptr;  // ncclComm_t
  int nranks = 1, rank = 0, device = 0;
  // host-transport variant (sr_comm_create_host): the caller's all-gather
  sr_allgather_fn host_fn = nullptr;
  void* host_user = nullptr;
};
Comm* comm_create_host(int nranks, int rank, int device, sr_allgather_fn fn, void* user);
void nccl_unique_id(uint8_t out[128]);
Comm* comm_create(int nranks, int rank, const uint8_t id[128], int device);
void comm_destroy(Comm* c);
void nccl_allgather_bytes(Comm* c, const void* send, void* recv, size_t bytes, cudaStream_t s);

}  // namespace srh
