/*
 * semrank_b200.h — C-ABI of the B200-native prefill relevance ranker.
 *
 * Drop-in boundary for the reference scorer path (reference = semrank C++,
 * /root/reference/proj). Every entry point cites the reference interface it
 * replaces. Plain pointers and sizes only; no C++ or torch types cross it.
 * A C++ facade with the reference's own type names (semrank::ModelConfig,
 * ScoreRequest, ScoreResult, ScoringEngine) lives in semrank_b200.hpp.
 *
 * Conventions
 *   - Every function returns an sr_status (0 = OK). On failure a thread-local
 *     message is available from sr_last_error().
 *   - Host buffers are borrowed for the duration of the call and never kept.
 *   - One engine = one device + one CUDA stream; calls on one engine are
 *     serialised (ScoringEngine::score holds a mutex, engine.cpp:389-392).
 *   - There is no CPU fallback: scoring needs an sm_100 device and fails with
 *     SR_CUDA otherwise.
 */
#ifndef SEMRANK_B200_H_
#define SEMRANK_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SR_ABI_VERSION 2  /* 2: sr_sched_stats gained max_pass_ms / max_wait_ms, sr_sched_options sat_rows; sr_engine_reserve */

/* Status codes. 1..15 mirror semrank::ErrorCode in declaration order
 * (include/semrank/error.hpp:13-29) so a facade can rethrow
 * semrank::Error{ErrorCode(status - 1)}. */
typedef enum sr_status {
  SR_OK = 0,
  SR_LENGTH_OVERFLOW = 1,
  SR_MASK_INVALID = 2,
  SR_SPEC_VIOLATION = 3,
  SR_PAYLOAD_INVALID = 4,
  SR_SCHEMA_UNKNOWN = 5,
  SR_ALIGNMENT = 6,
  SR_DIVERGENCE = 7,
  SR_PARAMETER = 8,
  SR_DEGENERATE_INPUT = 9,
  SR_UNDEFINED_METRIC = 10,
  SR_STATE_INVALID = 11,
  SR_OVERSIZE_ITEM = 12,
  SR_CONSISTENCY = 13,
  SR_RECONCILIATION = 14,
  SR_IO = 15,
  SR_CUDA = 100,
  SR_NCCL = 101
} sr_status;

/* ScoreMode (engine.hpp:15). */
typedef enum sr_score_mode {
  SR_MODE_NAIVE = 0,
  SR_MODE_IBPC = 1,
  SR_MODE_MULTI_ITEM = 2,
  SR_MODE_MIXED = 3
} sr_score_mode;

/* Mixed-mode items given as compact per-item embeddings (sr_engine_score_emb). */
typedef enum sr_emb_form {
  SR_EMB_PAD = 0,     /* one soft row per item: the embedding zero-padded (or cut) to
                         d_model, as SearchService::handle_search and cmd_score build
                         mixed items (service.cpp:208-217, semrank_main.cpp:362-368) */
  SR_EMB_PROJECT = 1  /* n_soft rows per item = emb . P (sr_engine_set_projection) */
} sr_emb_form;

/* Weight-init schemes for sr_weights_init. */
typedef enum sr_init_scheme {
  SR_INIT_REFERENCE = 0, /* init_model (model.cpp:94-134): N(0, 0.08^2) clamped to +-1 */
  SR_INIT_FAN_IN = 1     /* same stream/order, std 1/sqrt(fan_in), residual outputs /sqrt(2L) */
} sr_init_scheme;

/* ModelConfig (model.hpp:24-40). head_names/head_arity have n_task_heads
 * entries (HeadSpec, model.hpp:16-19). */
typedef struct sr_model_config {
  int32_t n_layers;
  int32_t d_model;
  int32_t n_heads;
  int32_t d_ff;
  int32_t vocab_size;
  int32_t max_seq;
  int32_t yes_token_id;
  int32_t no_token_id;
  int32_t n_task_heads;
  const char* const* head_names;
  const int32_t* head_arity;
} sr_model_config;

/* FlopReport (engine.hpp:38-44). */
typedef struct sr_flop_report {
  double attention_units;
  double linear_units;
  double t_q;
  double t_i_mean;
  double n_items;
} sr_flop_report;

/* ScoreRequest / ScoreItem (engine.hpp:20-33), flattened.
 *   token modes: item i = item_tokens[item_offsets[i] .. item_offsets[i+1])
 *   mixed mode : item i = item_rows[item_offsets[i]*d .. item_offsets[i+1]*d)
 *                ([n_emb_tokens x d_model] fp32 soft-token rows)
 * item_ids may be NULL (ids = 0..n_items-1); they are the doc ids used by the
 * top-k tie rule (score desc, doc_id asc). */
typedef struct sr_request {
  const int32_t* prefix_tokens;
  int32_t t_q;
  int32_t n_items;
  const int32_t* item_offsets; /* [n_items + 1], item_offsets[0] == 0 */
  const int32_t* item_tokens;
  const float* item_rows;
  const int64_t* item_ids;
  int32_t mode; /* sr_score_mode */
} sr_request;

/* ScoreResult (engine.hpp:53-59) plus the caller-side top-k. Any output
 * pointer may be NULL. scores is [n_items x n_tasks] with column 0 =
 * relevance and columns 1.. = task heads in config order (sr_task_count). */
typedef struct sr_result {
  double* scores;
  int32_t k;            /* top-k length requested (0 = none) */
  int64_t* topk_ids;    /* [k] */
  double* topk_scores;  /* [k] relevance */
  int32_t* topk_index;  /* [k] position in the request's item list */
  sr_flop_report flops; /* filled on success */
  double kv_incremental_per_item;
  int32_t k_returned;   /* min(k, n_items) */
} sr_result;

typedef struct sr_weights sr_weights;
typedef struct sr_engine sr_engine;
typedef struct sr_comm sr_comm;
typedef struct sr_plan sr_plan;
typedef struct sr_corpus sr_corpus;
typedef struct sr_wire sr_wire;

/* ------------------------------------------------------------ diagnostics */
const char* sr_last_error(void);
/* error_code_name (error.cpp:8-27) for 1..15, "cuda"/"nccl"/"ok" otherwise. */
const char* sr_status_name(int32_t status);
int32_t sr_abi_version(void);

/* ------------------------------------------------- host-side (no GPU needed) */
/* ModelConfig::validate (model.cpp:29-50). */
int32_t sr_config_validate(const sr_model_config* cfg);
/* ModelConfig::default_toy (model.cpp:52-57). Pointers inside are static. */
void sr_config_default_toy(sr_model_config* out);
/* 1 (relevance) + number of task heads. */
int32_t sr_task_count(const sr_model_config* cfg);

/* ModelWeights (model.hpp:56-67) on the host. Tensors are in the SRNKWTS1
 * canonical order (weights_io.cpp:47-71). */
int32_t sr_weights_init(const sr_model_config* cfg, uint64_t seed, int32_t scheme,
                        sr_weights** out); /* init_model, model.cpp:94-134 */
int32_t sr_weights_load(const char* path, sr_weights** out);         /* weights_io.cpp:137-196 */
int32_t sr_weights_save(const sr_weights* w, const char* path);      /* weights_io.cpp:104-135 */
int32_t sr_weights_from_tensors(const sr_model_config* cfg, const char* version,
                                const float* const* tensors, sr_weights** out);
void sr_weights_free(sr_weights* w);
/* Config view; pointers stay valid while w lives. */
int32_t sr_weights_config(const sr_weights* w, sr_model_config* out);
const char* sr_weights_version(const sr_weights* w);
size_t sr_weights_tensor_count(const sr_weights* w);
int32_t sr_weights_tensor(const sr_weights* w, size_t i, const char** name, float** data,
                          size_t* numel);

/* flops (engine.cpp:30-47). */
int32_t sr_flops(int32_t mode, int64_t t_q, int64_t t_i, int64_t n_items, sr_flop_report* out);
/* MultiItemMask::allowed_pair_count (engine.cpp:147-155). */
int32_t sr_multi_item_pair_count(int32_t prefix_len, const int32_t* item_lengths, int32_t n,
                                 int64_t* out);
/* build_multi_item_mask + to_attention_mask (engine.cpp:157-184): per packed
 * item row, {prefix_end, span_start} pairs (2 ints per row). */
int32_t sr_multi_item_mask(int32_t prefix_len, const int32_t* item_lengths, int32_t n,
                           int32_t* entries_out, int32_t cap_rows, int32_t* n_rows_out);
/* plan_batches (engine.cpp:278-326). requests given as prefix lengths and
 * flattened per-request item lengths (req_item_off[r]..req_item_off[r+1]).
 * Output entries: (batch, request_index, item_begin, item_end) quadruples. */
int32_t sr_plan_batches(int32_t n_requests, const int32_t* prefix_len,
                        const int32_t* req_item_off, const int32_t* item_len,
                        int64_t max_batch_tokens, int32_t* entries_out, int32_t cap_entries,
                        int32_t* n_entries_out, int64_t* batch_tokens_out, int32_t cap_batches,
                        int32_t* n_batches_out);
/* Validates a request against a config exactly as scoring would (same error
 * categories: engine.cpp:51-61, 243-251; model.cpp:222-264) and returns the
 * FlopReport / kv_incremental_per_item the reference reports for its mode. */
int32_t sr_request_report(const sr_model_config* cfg, const sr_request* req,
                          sr_flop_report* flops_out, double* kv_out);
/* Host top-k with the caller comparator (score desc, id asc, index asc). */
int32_t sr_topk_host(const double* scores, const int64_t* ids, int32_t n, int32_t k,
                     int64_t* ids_out, double* scores_out, int32_t* index_out);

/* build_prompt (prompt.cpp:14-38, prompt.hpp:17-25): prefix = system +
 * query_context, item = document + "\nRelevant (Yes/No): ", both byte-
 * tokenised (tokenizer.cpp:10-20). SR_LENGTH_OVERFLOW when the two exceed
 * max_seq, then SR_SPEC_VIOLATION for an empty prefix (the reference's
 * order and messages). Writes up to *_cap tokens; *n_prefix / *n_item get the
 * full lengths (call with cap 0 to size the buffers). */
int32_t sr_build_prompt(const char* system, int64_t system_len, const char* query_context,
                        int64_t query_len, const char* document, int64_t document_len,
                        int32_t max_seq, int32_t* prefix_out, int32_t prefix_cap,
                        int32_t* n_prefix, int32_t* item_out, int32_t item_cap, int32_t* n_item);
/* score_result_to_json (service.cpp:380-391), the /score response body, byte
 * for byte as the reference's nlohmann::json dump(): {"flops":{"attention",
 * "linear"},"request_id","scores":[{"id","tasks":{name: p, ...}}]} with keys
 * sorted. scores is [n_items x n_tasks] (sr_result.scores layout), column t
 * named task_names[t]. Writes up to cap bytes (no terminator); *len = full
 * length. SR_PAYLOAD_INVALID for ids/names that are not valid UTF-8. */
int32_t sr_score_result_to_json(const char* request_id, int32_t n_items,
                                const char* const* item_ids, int32_t n_tasks,
                                const char* const* task_names, const double* scores,
                                const sr_flop_report* flops, char* out, int64_t cap,
                                int64_t* len);

/* ------------------------------------------------------------------ engine */
/* ScoringEngine(const ModelWeights&) (engine.hpp:109-119), bound to a device:
 * converts the GEMM weights to bf16 K-major on the device once. */
int32_t sr_engine_create(const sr_weights* w, int32_t device, sr_engine** out);
void sr_engine_destroy(sr_engine* e);
/* ScoringEngine::score / score_by_mode (engine.cpp:379-392) + top-k. */
int32_t sr_engine_score(sr_engine* e, const sr_request* req, sr_result* res);
/* Batched multi-query scoring (plan_batches generalisation): n_req requests
 * packed into one device pass; res[i] receives request i's result. */
int32_t sr_engine_score_batch(sr_engine* e, const sr_request* reqs, int32_t n_req,
                              sr_result* res);
/* Debug/parity: final-LN hidden row at each item's last position
 * ([n_items x d_model] fp32), i.e. the row task_scores() consumes. */
int32_t sr_engine_item_hidden(sr_engine* e, const sr_request* req, float* hidden_out);
/* Context compression with precomputed item embeddings (north_star (d);
 * the reference injects d_model-wide rows only). P is the
 * projection in the reference's weight layout [d_emb x n_soft*d_model]
 * (row-major, model.hpp:42-47); item i's soft rows are
 *   rows_i = reshape(bf16(emb_i) . bf16(P), [n_soft x d_model])
 * computed on the tensor cores with fp32 accumulation inside the forward, so
 * only [n x d_emb] floats cross PCIe. proj == NULL removes it. */
int32_t sr_engine_set_projection(sr_engine* e, const float* proj, int32_t d_emb, int32_t n_soft);
/* Scores items given as emb [n_items x d_emb] fp32 (row-major) in mixed mode
 * (score_mixed, engine.cpp:238-276) with the rows of `form` (sr_emb_form).
 * SR_STATE_INVALID for SR_EMB_PROJECT without a projection, SR_ALIGNMENT when
 * d_emb differs from the projection's, SR_PAYLOAD_INVALID for no items or
 * d_emb < 1. FlopReport / kv as score_mixed with 1 or n_soft rows per item. */
int32_t sr_engine_score_emb(sr_engine* e, const int32_t* prefix, int32_t t_q, const float* emb,
                            int32_t d_emb, int32_t n_items, const int64_t* item_ids,
                            int32_t form, sr_result* res);
/* Sizes the engine's packed-row workspace for passes of up to `rows` rows
 * (prefix + item tokens summed over a pass's requests). Growing the workspace
 * invalidates every captured pass graph (each is re-captured on its next run),
 * so a server reserves its largest pass once, before it warms its pass
 * shapes; later passes that fit never move it. SR_PARAMETER for rows < 1 or
 * rows > 2^29. No reference counterpart (the reference has no device
 * workspace); serving-side addition next to ScoringEngine (engine.hpp:91-103). */
int32_t sr_engine_reserve(sr_engine* e, int64_t rows);
/* Device / stream the engine runs on. */
int32_t sr_engine_device(const sr_engine* e);
void* sr_engine_stream(const sr_engine* e);

/* Resident-input path (benchmarking / serving loops): a plan owns packed
 * device inputs and a captured CUDA graph for one request shape. */
int32_t sr_plan_create(sr_engine* e, const sr_request* req, int32_t k, sr_plan** out);
/* Several requests packed into one resident pass (per-request top-k). */
int32_t sr_plan_create_batch(sr_engine* e, const sr_request* reqs, int32_t n_req, int32_t k,
                             sr_plan** out);
/* Resident compact-embedding request (sr_engine_score_emb's inputs); the
 * pad / projection step is part of the plan's graph. */
int32_t sr_plan_create_emb(sr_engine* e, const int32_t* prefix, int32_t t_q, const float* emb,
                           int32_t d_emb, int32_t n_items, const int64_t* item_ids, int32_t form,
                           int32_t k, sr_plan** out);
/* Results of a batch plan: res[i] receives request i. */
int32_t sr_plan_fetch_batch(sr_plan* p, sr_result* res, int32_t n_req);
int32_t sr_plan_run(sr_plan* p);         /* enqueue on the engine stream; async */
int32_t sr_plan_sync(sr_plan* p);
int32_t sr_plan_fetch(sr_plan* p, sr_result* res); /* D2H of scores + top-k */
int32_t sr_plan_kernel_count(const sr_plan* p, int32_t* launches);
void sr_plan_destroy(sr_plan* p);
/* Live per-kernel-class timing: eager forward with CUDA events around each
 * launch on the engine stream. Classes: 0 embed+LN1, 1 QKV GEMM, 2 attention,
 * 3 O GEMM, 4 LayerNorm, 5 W_in GEMM, 6 W_out GEMM, 7 score head, 8 top-k.
 * ms_out[9] = mean ms per forward; launches_out[9] = launches per forward. */
#define SR_PROF_CLASSES 9
int32_t sr_plan_profile(sr_plan* p, int32_t reps, float* ms_out, int32_t* launches_out);
/* Shape of a plan: {rows M, items, attention tiles, soft rows, H2D bytes per
 * call, D2H bytes per call, k, tasks}. */
int32_t sr_plan_shape(const sr_plan* p, int64_t* out8);

/* ------------------------------- serving scheduler
 * Latency-bounded dynamic batching in front of one engine. Callers submit
 * whole requests from any thread (deep-copied at submit unless borrow is set, validated with the
 * scoring error categories); one dispatcher thread packs the queued requests
 * FIFO into device passes — the greedy rule of plan_batches
 * (engine.cpp:278-326) over whole requests under max_rows, at most
 * max_queries per pass and, with budget_ms > 0, only while
 * age(oldest) + est_ms(rows) <= budget_ms (est learned from the passes run) —
 * and completes each ticket. Replaces callers queueing on ScoringEngine's
 * mutex (engine.cpp:389-392). Latency = submit -> completion (host clock:
 * queueing, H2D, device pass, D2H); p50/p99 by nearest rank as the
 * service's percentile_of (service.cpp:28-34). */
typedef struct sr_sched sr_sched;
typedef struct sr_sched_options {
  int32_t max_queries; /* >= 1 */
  int64_t max_rows;    /* packed-row budget per pass (>= 1) */
  double budget_ms;    /* latency rule (0 = off) */
  int32_t max_wait_us; /* an unfilled pass waits this long after its oldest arrival (0 = no wait) */
  int32_t k;           /* top-k per request */
  int32_t borrow;      /* nonzero: request arrays are borrowed until sr_sched_wait
                          returns (no copy at submit) */
  int64_t sat_rows;    /* a request of at least this many packed rows runs in a
                          pass of its own (it saturates the device alone:
                          batching it adds latency, not throughput); 0 = off */
} sr_sched_options;
typedef struct sr_sched_stats {
  int64_t submitted, completed, failed, batches;
  double mean_batch, p50_ms, p99_ms, max_ms, mean_ms;
  double ms_per_row; /* current pass-time estimate */
  double busy_ms;    /* summed pass durations */
  double max_pass_ms;   /* longest pass */
  double max_wait_ms;   /* longest queue wait (submit -> pass start) */
} sr_sched_stats;
/* One pass over n_req requests (tests: a host stand-in for the engine). */
typedef int32_t (*sr_sched_exec_fn)(const sr_request* reqs, int32_t n_req, sr_result* res,
                                    void* user);
int32_t sr_sched_create(sr_engine* e, const sr_sched_options* opt, sr_sched** out);
int32_t sr_sched_create_host(const sr_model_config* cfg, const sr_sched_options* opt,
                             sr_sched_exec_fn fn, void* user, sr_sched** out);
int32_t sr_sched_submit(sr_sched* s, const sr_request* req, uint64_t* ticket);
/* Blocks until the ticket completes; res as sr_engine_score (caller buffers,
 * k <= options.k). Returns the request's own status. */
int32_t sr_sched_wait(sr_sched* s, uint64_t ticket, sr_result* res, double* latency_ms,
                      int32_t* batch_queries);
/* Counters and latency percentiles since the last reset. */
int32_t sr_sched_get_stats(sr_sched* s, int32_t reset, sr_sched_stats* out);
/* Fails still-queued tickets with SR_STATE_INVALID, joins the dispatcher. */
void sr_sched_destroy(sr_sched* s);

/* ------------------------------------------------------- multi-GPU (NCCL) */
/* Candidate sharding: every rank holds the full weights, scores its shard
 * of the items (with global item ids) and the per-rank top-k lists are merged
 * with one ncclAllGather; every rank returns the global top-k. */
int32_t sr_nccl_unique_id(uint8_t out[128]);
int32_t sr_comm_create(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t device,
                       sr_comm** out);
/* Same candidate sharding with the per-rank top-k exchange (k x 24-byte
 * entries) carried by the caller's all-gather instead of NCCL — for
 * transports such as gloo/MPI, or several ranks sharing one device where NCCL
 * refuses duplicate GPUs. fn(send, recv, bytes, user) must write every rank's
 * `bytes` in rank order into recv and return 0. The local pass, sentinel
 * padding and the device merge are the NCCL path's. */
typedef int32_t (*sr_allgather_fn)(const void* send, void* recv, size_t bytes_per_rank,
                                   void* user);
int32_t sr_comm_create_host(int32_t nranks, int32_t rank, int32_t device, sr_allgather_fn fn,
                            void* user, sr_comm** out);
void sr_comm_destroy(sr_comm* c);
int32_t sr_engine_score_sharded(sr_engine* e, sr_comm* c, const sr_request* local_shard,
                                sr_result* res);
int32_t sr_plan_run_sharded(sr_plan* p, sr_comm* c); /* resident variant */

/* --------------------------------------- /score wire ingest
 * parse_score_request_json's embedding_b64 items (service.cpp:361-370):
 * n_items base64 float32 payloads, concatenated in text with char offsets
 * char_off[n_items + 1], are copied to HBM and decoded there (base64.cpp:
 * 60-108 semantics) straight into the soft-token rows, then scored in mixed
 * mode like sr_engine_score. SR_PAYLOAD_INVALID with the reference's
 * messages for the first failing item: length not a multiple of 4,
 * misplaced padding, invalid character, not whole float32 values, not
 * [n x d_model]. */
int32_t sr_engine_score_b64(sr_engine* e, const int32_t* prefix, int32_t t_q, const char* text,
                            const int64_t* char_off, int32_t n_items, const int64_t* item_ids,
                            sr_result* res);

/* Native /score body parser (parse_score_request_json, service.cpp:326-372):
 * one pass over the JSON; embedding_b64 payloads stay spans into `body`
 * (which must outlive the handle) and are decoded on the device by
 * sr_engine_score_wire. Errors as the reference (SR_PAYLOAD_INVALID,
 * SR_LENGTH_OVERFLOW for text > max_seq, SR_PARAMETER for an unknown mode).
 * Item ids that are all integers become the top-k doc ids. */
int32_t sr_wire_parse(const char* body, int64_t len, int32_t max_seq, sr_wire** out);
void sr_wire_destroy(sr_wire* w);
int32_t sr_wire_info(const sr_wire* w, int32_t* n_items, int32_t* mode, int32_t* t_q);
const char* sr_wire_request_id(const sr_wire* w);
const char* sr_wire_item_id(const sr_wire* w, int32_t i);
int32_t sr_engine_score_wire(sr_engine* e, const sr_wire* w, sr_result* res);

/* ------------------------------ service post-processing
 * The step after scoring in SearchService::handle_search (service.cpp:242-277):
 * calibrate() of the relevance with the fitted isotonic head
 * (calibration.hpp:17-33, calibration.cpp:65-88: blocks sorted by lo, value
 * clamped to [0,1], linear ramp across gaps), then the final score is the
 * calibrated relevance, or sum_j blend_w[j] * calibrated[blend_task[j]] in the
 * given order (the std::map<string,double> score_blend iterates by task name;
 * task 0 = relevance, 1.. = heads in config order). The device computes it in
 * the same double operation order and the top-k (page) orders by it; the
 * returned topk_scores are then final scores. n_blocks = n_blend = 0 turns
 * it off. SR_ALIGNMENT for an unknown blend task (service.cpp:258-262). */
int32_t sr_engine_set_postprocess(sr_engine* e, const double* lo, const double* hi,
                                  const double* value, int32_t n_blocks,
                                  const int32_t* blend_task, const double* blend_w,
                                  int32_t n_blend);
/* Final scores [n_items] of the last score call (post-processing on). */
int32_t sr_engine_final_scores(sr_engine* e, double* out, int32_t cap, int32_t* n_out);

/* Deterministic score cache (midtier.hpp:16-69, midtier.cpp:14-100; probed
 * and filled by SearchService::handle_search, service.cpp:160-234). Keys are
 * (searcher_id, query_signature, entity_id, model_version); LRU over whole
 * entries, get refreshes recency, a miss mutates nothing, put of a different
 * row under an existing key is SR_CONSISTENCY, capacity 0 is SR_PARAMETER.
 * Values are the engine's score rows (n_tasks doubles, column order as
 * sr_result.scores). Thread-safe (one mutex). */
typedef struct sr_score_cache sr_score_cache;
int32_t sr_score_cache_create(int64_t capacity, sr_score_cache** out);
void sr_score_cache_destroy(sr_score_cache* c);
int64_t sr_score_cache_size(const sr_score_cache* c);
int64_t sr_score_cache_capacity(const sr_score_cache* c);
int32_t sr_score_cache_get(sr_score_cache* c, const char* searcher_id, uint64_t query_signature,
                           int64_t entity_id, const char* model_version, double* scores,
                           int32_t n_tasks, int32_t* hit);
int32_t sr_score_cache_put(sr_score_cache* c, const char* searcher_id, uint64_t query_signature,
                           int64_t entity_id, const char* model_version, const double* scores,
                           int32_t n_tasks);
/* canonical_query (midtier.cpp:14-44): lowercased, whitespace runs collapsed
 * and trimmed, then "|attr=v1,v2" per attribute (byte order, values sorted).
 * Filters are n_filters (attrs[i], values[i]) pairs; a repeated attr
 * collects its values. Writes up to cap bytes (no terminator) and the full
 * length to *len. sr_query_signature = fnv1a64(canonical_query(...)). */
int32_t sr_canonical_query(const char* text, int32_t n_filters, const char* const* attrs,
                           const char* const* values, char* out, int64_t cap, int64_t* len);
int32_t sr_query_signature(const char* text, int32_t n_filters, const char* const* attrs,
                           const char* const* values, uint64_t* out);
uint64_t sr_fnv1a64(const char* data, int64_t len); /* midtier.cpp:46-53 */
/* handle_search's cache path (service.cpp:160-234) around the device scorer:
 * probe every item (req->item_ids = entity ids), score only the misses in
 * one forward pass (request order), put their rows, then rank all rows on
 * the device (post-processing when set, top-k by (key desc, id asc)).
 * res->scores receives all rows; *n_hits the cache hits. flops describe the
 * miss pass (zero when everything hit). */
int32_t sr_engine_score_cached(sr_engine* e, sr_score_cache* c, const char* searcher_id,
                               uint64_t query_signature, const char* model_version,
                               const sr_request* req, sr_result* res, int32_t* n_hits);

/* ------------------------------- exhaustive retrieval top-K
 * The candidate generator upstream of the ranker. Replaces
 *   std::vector<RankedDoc> exhaustive_topk(const Corpus&, const QuerySpec&,
 *                                          const RARWeights&, kernels::Exec)
 * (retrieval.hpp:60-70, retrieval.cpp:134-173) with rar_score (:60-71) and
 * cosine (:44-58): S = w0 cos(q, e_d) + sum_i w_i f_i(d), exact top-K by
 * (score desc, doc_id asc), scores bit-identical to the reference's doubles.
 * Corpus (retrieval.hpp:21-33) is passed columnar: embeddings [n x d_emb],
 * features [n x n_features] in feature_names order, doc ids [n]; it is
 * copied to the device once. QuerySpec.filters are applied by the caller as
 * a keep mask (filter_candidates, retrieval.cpp:79-97; NULL = all docs).
 * Errors as the reference: SR_SPEC_VIOLATION (k < 1), SR_ALIGNMENT (weight
 * count or query dimension mismatch), SR_DEGENERATE_INPUT (zero query or
 * document vector among the candidates); no checks run without candidates. */
int32_t sr_corpus_create(const float* embeddings, const float* features, const int64_t* doc_ids,
                         int64_t n_docs, int32_t d_emb, int32_t n_features, int32_t device,
                         sr_corpus** out);
void sr_corpus_destroy(sr_corpus* c);
/* Writes min(k, #candidates) entries; *n_out = that count. */
int32_t sr_corpus_topk(sr_corpus* c, const float* query, int32_t d_query, double w0,
                       const double* w, int32_t n_w, const uint8_t* keep, int32_t k,
                       int64_t* ids_out, double* scores_out, int32_t* n_out);
/* This rank holds a shard of the corpus (global doc ids); one NCCL
 * all-gather of k entries per rank + the comparator merge (the reference's
 * shard merge, retrieval.cpp:144-165) gives every rank the global top-K. */
int32_t sr_corpus_topk_sharded(sr_corpus* c, sr_comm* comm, const float* query, int32_t d_query,
                               double w0, const double* w, int32_t n_w, const uint8_t* keep,
                               int32_t k, int64_t* ids_out, double* scores_out, int32_t* n_out);
/* Docs rescored in double by the last call (the fp32 pass's candidate set). */
int64_t sr_corpus_last_candidates(const sr_corpus* c);
/* Device time (ms, CUDA events on the corpus stream) of the last call's
 * fp32 scan kernel (the HBM-bound pass; bench roofline). */
float sr_corpus_last_scan_ms(const sr_corpus* c);

/* --------------------------------------- kernel-level entry points (tests) */
/* All pointers are device pointers; stream may be NULL (legacy stream). */
/* C[M x N] = A[M x K] . B[N x K]^T ; epi 0 bf16, 1 gelu->bf16, 2 fp32 C += acc, 3 fp32.
 * Synchronous when stream is NULL, asynchronous on an explicit stream. */
int32_t sr_kernel_gemm(const void* a_bf16, const void* b_bf16, int32_t M, int32_t N, int32_t K,
                       void* c, int32_t ldc, int32_t epi, void* stream);
/* LayerNorm folded into the projections. Device pointers.
 * epi 4: c = x fp32 [M x N] += A.B^T, xb = bf16(x) [M x N],
 *        stats[N/128][ld] = float2 (mean, M2) of x over each 128-column slice.
 * epi 5 / 6: c = bf16([gelu](rstd * (A.B^T - mean * colsum))), A = bf16 x,
 *        B = diag(gain) W, mean/rstd from stats[n_parts][ld] (each part over
 *        K / n_parts columns), colsum[N]. N % 256 == 0 (CTA-pair kernel). */
int32_t sr_kernel_gemm_ln(const void* a_bf16, const void* b_bf16, int32_t M, int32_t N, int32_t K,
                          void* c, int32_t ldc, int32_t epi, void* xb_bf16, void* stats,
                          int32_t n_parts, const float* colsum, int32_t ld, void* stream);
/* Residual projection with the next LayerNorm overlapped:
 * x fp32 [M x N] += A.B^T (GEMM epilogue 7 counts completed 128-row blocks)
 * while a concurrent kernel writes out_bf16 [M x N] = bf16(LN(x) * gain)
 * (kernels.cpp:31-45) block by block. counters: device uint32
 * [ceil(M / 128)], zero on entry and on return. N % 256 == 0, N <= 2048.
 * Device pointers; synchronous. */
int32_t sr_kernel_gemm_resid_ln(const void* a_bf16, const void* b_bf16, int32_t M, int32_t N,
                                int32_t K, float* x, const float* gain, void* out_bf16,
                                uint32_t* counters, void* stream);
/* Segment-masked attention. qkv [M x 3d] bf16, spans [M x 4] int32
 * {prefix_begin, prefix_end, span_start, 0}; out [M x d] bf16. Tiles are
 * planned internally. */
int32_t sr_kernel_attention(const void* qkv, const int32_t* spans_host, int32_t M,
                            int32_t n_heads, int32_t head_dim, void* out, void* stream);
int32_t sr_kernel_layernorm(const float* x, const float* gain, void* out_bf16, int32_t M,
                            int32_t d, void* stream);
/* Tuning aid: record a clock64 timeline (64 slots per CTA, first 256 tiles of
 * head 0) from the tcgen05 attention kernel into dev_buf; NULL disables. */
int32_t sr_debug_attention_trace(void* dev_buf);
/* Tuning aid: %globaltimer timeline of the CTA-pair GEMM (64 slots per CTA). */
int32_t sr_debug_gemm_trace(void* dev_buf);
int32_t sr_kernel_topk(const double* scores, const int64_t* ids, int32_t n, int32_t k,
                       int64_t* ids_out_host, double* scores_out_host, int32_t* index_out_host);

#ifdef __cplusplus
}
#endif

#endif /* SEMRANK_B200_H_ */
