// extern "C" boundary (include/semrank_b200.h): thin wrappers that map
// srh::Error to sr_status and keep a thread-local error message.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "host/engine.hpp"
#include "host/retrieval.hpp"
#include "host/score_cache.hpp"
#include "host/wire.hpp"
#include "host/model.hpp"
#include "host/planner.hpp"
#include "host/prompt.hpp"
#include "host/scheduler.hpp"
#include "kernels/launch.h"
#include "semrank_b200.h"

namespace srh {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace srh

using srh::guard;

struct sr_weights {
  srh::ModelWeights w;
  std::vector<std::string> head_name_store;
  std::vector<const char*> head_names;
  std::vector<int32_t> head_arity;
  std::vector<std::pair<std::string, std::vector<float>*>> table;
  void refresh() {
    head_name_store.clear();
    head_names.clear();
    head_arity.clear();
    for (const auto& h : w.config.head_specs) {
      head_name_store.push_back(h.name);
      head_arity.push_back(h.arity);
    }
    for (const auto& s : head_name_store) head_names.push_back(s.c_str());
    table = w.tensor_table();
  }
};

struct sr_engine {
  std::unique_ptr<srh::Engine> e;
};

struct sr_comm {
  srh::Comm* c = nullptr;
};

struct sr_wire {
  srh::WireRequest w;
  std::vector<int64_t> ids;  // item ids as doc ids when every id is an integer
  bool numeric_ids = false;
};

struct sr_score_cache {
  std::unique_ptr<srh::ScoreCache> c;
};

struct sr_corpus {
  std::unique_ptr<srh::Corpus> c;
  std::mutex mu;  // one scan at a time per corpus (one stream)
};

struct sr_plan {
  sr_engine* owner = nullptr;
  std::unique_ptr<srh::Plan> p;
  bool sharded_valid = false;
};

namespace {

void copy_topk_merged(srh::Plan& p, sr_result* res, cudaStream_t s) {
  std::vector<srk::TopkEntry> top(p.k);
  SR_CUDA_CHECK(cudaMemcpyAsync(top.data(), p.merged.ptr, top.size() * sizeof(srk::TopkEntry),
                                cudaMemcpyDeviceToHost, s));
  SR_CUDA_CHECK(cudaStreamSynchronize(s));
  int32_t kr = 0;
  for (int32_t j = 0; j < std::min(res->k, p.k); ++j) {
    const auto& e = top[j];
    if (e.index == INT32_MAX) break;  // sentinel: fewer candidates than k
    if (res->topk_ids) res->topk_ids[j] = e.id;
    if (res->topk_scores) res->topk_scores[j] = e.score;
    if (res->topk_index) res->topk_index[j] = -1;  // global: index is rank-local
    ++kr;
  }
  res->k_returned = kr;
}

}  // namespace

extern "C" {

const char* sr_last_error(void) { return srh::g_last_error.c_str(); }

const char* sr_status_name(int32_t status) {
  static const char* names[] = {"ok",
                                "length_overflow",
                                "mask_invalid",
                                "spec_violation",
                                "payload_invalid",
                                "schema_unknown",
                                "alignment",
                                "divergence",
                                "parameter",
                                "degenerate_input",
                                "undefined_metric",
                                "state_invalid",
                                "oversize_item",
                                "consistency",
                                "reconciliation",
                                "io"};
  if (status >= 0 && status <= 15) return names[status];
  if (status == SR_CUDA) return "cuda";
  if (status == SR_NCCL) return "nccl";
  return "unknown";
}

int32_t sr_abi_version(void) { return SR_ABI_VERSION; }

int32_t sr_config_validate(const sr_model_config* cfg) {
  return guard([&] {
    if (!cfg) srh::fail(SR_SPEC_VIOLATION, "null config");
    srh::ModelConfig::from_c(*cfg).validate();
  });
}

void sr_config_default_toy(sr_model_config* out) {
  static const char* names[] = {"click", "apply", "badfit", "shortlist", "dismiss"};
  static const int32_t arity[] = {1, 1, 1, 1, 1};
  out->n_layers = 2;
  out->d_model = 64;
  out->n_heads = 4;
  out->d_ff = 256;
  out->vocab_size = 300;
  out->max_seq = srh::kDefaultMaxSeq;
  out->yes_token_id = srh::kTokenYes;
  out->no_token_id = srh::kTokenNo;
  out->n_task_heads = 5;
  out->head_names = names;
  out->head_arity = arity;
}

int32_t sr_task_count(const sr_model_config* cfg) { return cfg ? 1 + cfg->n_task_heads : 0; }

int32_t sr_weights_init(const sr_model_config* cfg, uint64_t seed, int32_t scheme,
                        sr_weights** out) {
  return guard([&] {
    if (!cfg || !out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    auto w = std::make_unique<sr_weights>();
    w->w = srh::init_model(srh::ModelConfig::from_c(*cfg), seed, scheme);
    w->refresh();
    *out = w.release();
  });
}

int32_t sr_weights_load(const char* path, sr_weights** out) {
  return guard([&] {
    if (!path || !out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    auto w = std::make_unique<sr_weights>();
    w->w = srh::load_weights(path);
    w->refresh();
    *out = w.release();
  });
}

int32_t sr_weights_save(const sr_weights* w, const char* path) {
  return guard([&] {
    if (!w || !path) srh::fail(SR_SPEC_VIOLATION, "null argument");
    srh::save_weights(w->w, path);
  });
}

int32_t sr_weights_from_tensors(const sr_model_config* cfg, const char* version,
                                const float* const* tensors, sr_weights** out) {
  return guard([&] {
    if (!cfg || !tensors || !out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    auto w = std::make_unique<sr_weights>();
    w->w.config = srh::ModelConfig::from_c(*cfg);
    w->w.config.validate();
    w->w.version = version ? version : "";
    w->w.allocate();
    size_t i = 0;
    for (auto& [name, t] : w->w.tensor_table()) {
      if (!tensors[i]) srh::fail(SR_SPEC_VIOLATION, "null tensor " + name);
      std::memcpy(t->data(), tensors[i], t->size() * sizeof(float));
      ++i;
    }
    w->refresh();
    *out = w.release();
  });
}

void sr_weights_free(sr_weights* w) { delete w; }

int32_t sr_weights_config(const sr_weights* w, sr_model_config* out) {
  return guard([&] {
    if (!w || !out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    const auto& c = w->w.config;
    out->n_layers = c.n_layers;
    out->d_model = c.d_model;
    out->n_heads = c.n_heads;
    out->d_ff = c.d_ff;
    out->vocab_size = c.vocab_size;
    out->max_seq = c.max_seq;
    out->yes_token_id = c.yes_token_id;
    out->no_token_id = c.no_token_id;
    out->n_task_heads = static_cast<int32_t>(c.head_specs.size());
    out->head_names = w->head_names.data();
    out->head_arity = w->head_arity.data();
  });
}

const char* sr_weights_version(const sr_weights* w) { return w ? w->w.version.c_str() : ""; }

size_t sr_weights_tensor_count(const sr_weights* w) { return w ? w->table.size() : 0; }

int32_t sr_weights_tensor(const sr_weights* w, size_t i, const char** name, float** data,
                          size_t* numel) {
  return guard([&] {
    if (!w || i >= w->table.size()) srh::fail(SR_PARAMETER, "tensor index out of range");
    if (name) *name = w->table[i].first.c_str();
    if (data) *data = w->table[i].second->data();
    if (numel) *numel = w->table[i].second->size();
  });
}

int32_t sr_flops(int32_t mode, int64_t t_q, int64_t t_i, int64_t n_items, sr_flop_report* out) {
  return guard([&] {
    const auto r = srh::flops(mode, t_q, t_i, n_items);
    if (out) *out = r;
  });
}

int32_t sr_multi_item_pair_count(int32_t prefix_len, const int32_t* item_lengths, int32_t n,
                                 int64_t* out) {
  return guard([&] {
    if (prefix_len < 0) srh::fail(SR_SPEC_VIOLATION, "negative prefix length");
    for (int i = 0; i < n; ++i)
      if (item_lengths[i] < 1) srh::fail(SR_SPEC_VIOLATION, "zero-length item in multi-item mask");
    *out = srh::multi_item_pair_count(prefix_len, item_lengths, n);
  });
}

int32_t sr_multi_item_mask(int32_t prefix_len, const int32_t* item_lengths, int32_t n,
                           int32_t* entries_out, int32_t cap_rows, int32_t* n_rows_out) {
  return guard([&] {  // engine.cpp:157-184
    if (prefix_len < 0) srh::fail(SR_SPEC_VIOLATION, "negative prefix length");
    int32_t rows = 0, cursor = prefix_len;
    for (int i = 0; i < n; ++i) {
      const int32_t len = item_lengths[i];
      if (len < 1) srh::fail(SR_SPEC_VIOLATION, "zero-length item in multi-item mask");
      for (int32_t p = cursor; p < cursor + len; ++p, ++rows) {
        if (entries_out && rows < cap_rows) {
          entries_out[2 * rows] = prefix_len;
          entries_out[2 * rows + 1] = cursor;
        }
      }
      cursor += len;
    }
    if (n_rows_out) *n_rows_out = rows;
    if (entries_out && rows > cap_rows) srh::fail(SR_PARAMETER, "mask output buffer too small");
  });
}

int32_t sr_plan_batches(int32_t n_requests, const int32_t* prefix_len,
                        const int32_t* req_item_off, const int32_t* item_len,
                        int64_t max_batch_tokens, int32_t* entries_out, int32_t cap_entries,
                        int32_t* n_entries_out, int64_t* batch_tokens_out, int32_t cap_batches,
                        int32_t* n_batches_out) {
  return guard([&] {
    std::vector<int32_t> pl(prefix_len, prefix_len + n_requests);
    std::vector<std::vector<int32_t>> il(n_requests);
    for (int r = 0; r < n_requests; ++r)
      il[r].assign(item_len + req_item_off[r], item_len + req_item_off[r + 1]);
    const auto batches = srh::plan_batches(pl, il, max_batch_tokens);
    int32_t ne = 0;
    for (size_t b = 0; b < batches.size(); ++b) {
      if (batch_tokens_out && static_cast<int32_t>(b) < cap_batches)
        batch_tokens_out[b] = batches[b].token_count;
      for (const auto& e : batches[b].entries) {
        if (entries_out && ne < cap_entries) {
          entries_out[4 * ne + 0] = static_cast<int32_t>(b);
          entries_out[4 * ne + 1] = e.request_index;
          entries_out[4 * ne + 2] = e.item_begin;
          entries_out[4 * ne + 3] = e.item_end;
        }
        ++ne;
      }
    }
    if (n_entries_out) *n_entries_out = ne;
    if (n_batches_out) *n_batches_out = static_cast<int32_t>(batches.size());
    if ((entries_out && ne > cap_entries) ||
        (batch_tokens_out && static_cast<int32_t>(batches.size()) > cap_batches))
      srh::fail(SR_PARAMETER, "plan output buffers too small");
  });
}

int32_t sr_request_report(const sr_model_config* cfg, const sr_request* req,
                          sr_flop_report* flops_out, double* kv_out) {
  return guard([&] {
    if (!cfg || !req) srh::fail(SR_SPEC_VIOLATION, "null argument");
    const auto c = srh::ModelConfig::from_c(*cfg);
    c.validate();
    const auto lens = srh::validate_request(c, *req);
    srh::report_for(c, *req, lens, flops_out, kv_out);
  });
}

int32_t sr_topk_host(const double* scores, const int64_t* ids, int32_t n, int32_t k,
                     int64_t* ids_out, double* scores_out, int32_t* index_out) {
  return guard([&] {
    if (n < 0 || k < 0) srh::fail(SR_PARAMETER, "negative size");
    const auto top = srh::topk_host(scores, ids, n, k);
    for (size_t j = 0; j < top.size(); ++j) {
      if (ids_out) ids_out[j] = top[j].id;
      if (scores_out) scores_out[j] = top[j].score;
      if (index_out) index_out[j] = top[j].index;
    }
  });
}

int32_t sr_build_prompt(const char* system, int64_t system_len, const char* query_context,
                        int64_t query_len, const char* document, int64_t document_len,
                        int32_t max_seq, int32_t* prefix_out, int32_t prefix_cap,
                        int32_t* n_prefix, int32_t* item_out, int32_t item_cap, int32_t* n_item) {
  return guard([&] {
    if (system_len < 0 || query_len < 0 || document_len < 0 || prefix_cap < 0 || item_cap < 0)
      srh::fail(SR_PARAMETER, "negative size");
    if ((system_len && !system) || (query_len && !query_context) || (document_len && !document) ||
        !n_prefix || !n_item)
      srh::fail(SR_SPEC_VIOLATION, "null argument");
    const auto parts = srh::build_prompt(std::string_view(system ? system : "", system_len),
                                         std::string_view(query_context ? query_context : "", query_len),
                                         std::string_view(document ? document : "", document_len),
                                         max_seq);
    *n_prefix = static_cast<int32_t>(parts.prefix_tokens.size());
    *n_item = static_cast<int32_t>(parts.item_tokens.size());
    if (prefix_out)
      std::copy_n(parts.prefix_tokens.begin(), std::min<size_t>(prefix_cap, parts.prefix_tokens.size()),
                  prefix_out);
    if (item_out)
      std::copy_n(parts.item_tokens.begin(), std::min<size_t>(item_cap, parts.item_tokens.size()),
                  item_out);
  });
}

int32_t sr_score_result_to_json(const char* request_id, int32_t n_items,
                                const char* const* item_ids, int32_t n_tasks,
                                const char* const* task_names, const double* scores,
                                const sr_flop_report* flops, char* out, int64_t cap,
                                int64_t* len) {
  return guard([&] {
    if (n_items < 0 || n_tasks < 0 || cap < 0) srh::fail(SR_PARAMETER, "negative size");
    if (!len || !flops || (n_items > 0 && (!item_ids || (n_tasks > 0 && !scores))) ||
        (n_tasks > 0 && !task_names))
      srh::fail(SR_SPEC_VIOLATION, "null argument");
    for (int32_t t = 0; t < n_tasks; ++t)
      if (!task_names[t]) srh::fail(SR_SPEC_VIOLATION, "null task name");
    const std::string j = srh::score_result_json(request_id ? request_id : "", n_items, item_ids,
                                                 n_tasks, task_names, scores,
                                                 flops->attention_units, flops->linear_units);
    *len = static_cast<int64_t>(j.size());
    if (out) std::memcpy(out, j.data(), std::min<size_t>(static_cast<size_t>(cap), j.size()));
  });
}

int32_t sr_engine_create(const sr_weights* w, int32_t device, sr_engine** out) {
  return guard([&] {
    if (!w || !out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    auto e = std::make_unique<sr_engine>();
    e->e = std::make_unique<srh::Engine>(w->w, device);
    *out = e.release();
  });
}

void sr_engine_destroy(sr_engine* e) { delete e; }

int32_t sr_engine_score(sr_engine* e, const sr_request* req, sr_result* res) {
  return guard([&] {
    if (!e || !req || !res) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    e->e->score(req, 1, res);
  });
}

int32_t sr_engine_score_batch(sr_engine* e, const sr_request* reqs, int32_t n_req,
                              sr_result* res) {
  return guard([&] {
    if (!e || !reqs || !res) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    e->e->score(reqs, n_req, res);
  });
}

// ------------------------------------------------------------ scheduler
struct sr_sched {
  std::unique_ptr<srh::Scheduler> s;
};

static srh::SchedOptions sched_options(const sr_sched_options* o) {
  srh::SchedOptions so;
  if (o) {
    so.max_queries = o->max_queries;
    so.max_rows = o->max_rows;
    so.budget_ms = o->budget_ms;
    so.max_wait_us = o->max_wait_us;
    so.k = o->k;
    so.borrow = o->borrow != 0;
    so.sat_rows = o->sat_rows;
  }
  return so;
}

int32_t sr_sched_create(sr_engine* e, const sr_sched_options* opt, sr_sched** out) {
  return guard([&] {
    if (!e || !out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    srh::Engine* eng = e->e.get();
    auto s = std::make_unique<sr_sched>();
    s->s = std::make_unique<srh::Scheduler>(
        [eng](const sr_request* reqs, int n, sr_result* res) {
          std::lock_guard<std::mutex> lock(eng->mutex());
          eng->score(reqs, n, res);
        },
        eng->config(), sched_options(opt));
    *out = s.release();
  });
}

int32_t sr_sched_create_host(const sr_model_config* cfg, const sr_sched_options* opt,
                             sr_sched_exec_fn fn, void* user, sr_sched** out) {
  return guard([&] {
    if (!cfg || !fn || !out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    const auto c = srh::ModelConfig::from_c(*cfg);
    c.validate();
    auto s = std::make_unique<sr_sched>();
    s->s = std::make_unique<srh::Scheduler>(
        [fn, user](const sr_request* reqs, int n, sr_result* res) {
          const int32_t st = fn(reqs, n, res, user);
          if (st != SR_OK) srh::fail(static_cast<sr_status>(st), "scheduler pass failed");
        },
        c, sched_options(opt));
    *out = s.release();
  });
}

int32_t sr_sched_submit(sr_sched* s, const sr_request* req, uint64_t* ticket) {
  return guard([&] {
    if (!s || !req || !ticket) srh::fail(SR_SPEC_VIOLATION, "null argument");
    *ticket = s->s->submit(*req);
  });
}

int32_t sr_sched_wait(sr_sched* s, uint64_t ticket, sr_result* res, double* latency_ms,
                      int32_t* batch_queries) {
  return guard([&] {
    if (!s) srh::fail(SR_SPEC_VIOLATION, "null argument");
    s->s->wait(ticket, res, latency_ms, batch_queries);
  });
}

int32_t sr_sched_get_stats(sr_sched* s, int32_t reset, sr_sched_stats* out) {
  return guard([&] {
    if (!s || !out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    const srh::SchedStats st = s->s->stats(reset != 0);
    out->submitted = st.submitted;
    out->completed = st.completed;
    out->failed = st.failed;
    out->batches = st.batches;
    out->mean_batch = st.mean_batch;
    out->p50_ms = st.p50_ms;
    out->p99_ms = st.p99_ms;
    out->max_ms = st.max_ms;
    out->mean_ms = st.mean_ms;
    out->ms_per_row = st.ms_per_row;
    out->busy_ms = st.busy_ms;
    out->max_pass_ms = st.max_pass_ms;
    out->max_wait_ms = st.max_wait_ms;
  });
}

void sr_sched_destroy(sr_sched* s) { delete s; }

int32_t sr_engine_item_hidden(sr_engine* e, const sr_request* req, float* hidden_out) {
  return guard([&] {
    if (!e || !req || !hidden_out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    e->e->item_hidden(*req, hidden_out);
  });
}

int32_t sr_engine_score_b64(sr_engine* e, const int32_t* prefix, int32_t t_q, const char* text,
                            const int64_t* char_off, int32_t n_items, const int64_t* item_ids,
                            sr_result* res) {
  return guard([&] {
    if (!e || !res || !char_off || (t_q > 0 && !prefix) || (n_items > 0 && !text))
      srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    e->e->score_b64(prefix, t_q, text, char_off, n_items, item_ids, res);
  });
}

int32_t sr_wire_parse(const char* body, int64_t len, int32_t max_seq, sr_wire** out) {
  return guard([&] {
    if (!out || (len > 0 && !body)) srh::fail(SR_SPEC_VIOLATION, "null argument");
    auto w = std::make_unique<sr_wire>();
    w->w = srh::parse_wire(body, len, max_seq);
    w->numeric_ids = true;
    for (const auto& it : w->w.items) {
      char* endp = nullptr;
      const long long v = it.id.empty() ? 0 : std::strtoll(it.id.c_str(), &endp, 10);
      if (it.id.empty() || *endp != '\0') {
        w->numeric_ids = false;
        break;
      }
      w->ids.push_back(v);
    }
    if (!w->numeric_ids) w->ids.clear();
    *out = w.release();
  });
}

void sr_wire_destroy(sr_wire* w) { delete w; }

int32_t sr_wire_info(const sr_wire* w, int32_t* n_items, int32_t* mode, int32_t* t_q) {
  return guard([&] {
    if (!w) srh::fail(SR_SPEC_VIOLATION, "null argument");
    if (n_items) *n_items = static_cast<int32_t>(w->w.items.size());
    if (mode) *mode = w->w.mode;
    if (t_q) *t_q = static_cast<int32_t>(w->w.prefix.size());
  });
}

const char* sr_wire_request_id(const sr_wire* w) { return w ? w->w.request_id.c_str() : ""; }

const char* sr_wire_item_id(const sr_wire* w, int32_t i) {
  if (!w || i < 0 || i >= static_cast<int32_t>(w->w.items.size())) return "";
  return w->w.items[i].id.c_str();
}

int32_t sr_engine_score_wire(sr_engine* e, const sr_wire* w, sr_result* res) {
  return guard([&] {
    if (!e || !w || !res) srh::fail(SR_SPEC_VIOLATION, "null argument");
    const auto& r = w->w;
    const int32_t n = static_cast<int32_t>(r.items.size());
    const int64_t* ids = w->numeric_ids ? w->ids.data() : nullptr;
    std::lock_guard<std::mutex> lock(e->e->mutex());
    if (r.mode == SR_MODE_MIXED) {
      std::vector<int64_t> b(n), en(n);
      for (int32_t j = 0; j < n; ++j) {
        const auto& it = r.items[j];
        if (!it.b64)  // score_mixed needs an embedding per item (engine.cpp:243-251)
          srh::fail(SR_PAYLOAD_INVALID, "mixed request item without embedding_b64: " + it.id);
        const int64_t base = it.in_side ? r.body_len : 0;
        b[j] = base + it.b64_begin;
        en[j] = base + it.b64_end;
      }
      e->e->score_b64_spans(r.prefix.data(), static_cast<int32_t>(r.prefix.size()), r.body,
                            r.body_len, r.side.data(), static_cast<int64_t>(r.side.size()),
                            b.data(), en.data(), n, ids, res);
      return;
    }
    std::vector<int32_t> off(n + 1, 0), tok;
    for (int32_t j = 0; j < n; ++j) {
      tok.insert(tok.end(), r.items[j].tokens.begin(), r.items[j].tokens.end());
      off[j + 1] = static_cast<int32_t>(tok.size());
    }
    if (tok.empty()) tok.push_back(0);
    sr_request req{};
    req.prefix_tokens = r.prefix.data();
    req.t_q = static_cast<int32_t>(r.prefix.size());
    req.n_items = n;
    req.item_offsets = off.data();
    req.item_tokens = tok.data();
    req.item_rows = nullptr;
    req.item_ids = ids;
    req.mode = r.mode;
    e->e->score(&req, 1, res);
  });
}

int32_t sr_engine_set_postprocess(sr_engine* e, const double* lo, const double* hi,
                                  const double* value, int32_t n_blocks,
                                  const int32_t* blend_task, const double* blend_w,
                                  int32_t n_blend) {
  return guard([&] {
    if (!e || (n_blocks > 0 && (!lo || !hi || !value)) || (n_blend > 0 && (!blend_task || !blend_w)))
      srh::fail(SR_SPEC_VIOLATION, "null argument");
    // the blend weighs the calibrated relevance: an unfitted head throws
    // StateInvalid in the reference (calibration.cpp:65-68)
    if (n_blend > 0 && n_blocks <= 0)
      srh::fail(SR_STATE_INVALID, "calibration head not fitted");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    e->e->set_postprocess(lo, hi, value, n_blocks, blend_task, blend_w, n_blend);
  });
}

int32_t sr_engine_final_scores(sr_engine* e, double* out, int32_t cap, int32_t* n_out) {
  return guard([&] {
    if (!e || !n_out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    const auto& f = e->e->last_final();
    const int32_t n = static_cast<int32_t>(f.size());
    if (out)
      for (int32_t i = 0; i < std::min(n, cap); ++i) out[i] = f[i];
    *n_out = n;
  });
}

int32_t sr_score_cache_create(int64_t capacity, sr_score_cache** out) {
  return guard([&] {
    if (!out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    *out = nullptr;
    if (capacity < 0) srh::fail(SR_PARAMETER, "cache capacity must be >= 1");
    auto c = std::make_unique<sr_score_cache>();
    c->c = std::make_unique<srh::ScoreCache>(static_cast<size_t>(capacity));
    *out = c.release();
  });
}

void sr_score_cache_destroy(sr_score_cache* c) { delete c; }
int64_t sr_score_cache_size(const sr_score_cache* c) {
  return c ? static_cast<int64_t>(c->c->size()) : -1;
}
int64_t sr_score_cache_capacity(const sr_score_cache* c) {
  return c ? static_cast<int64_t>(c->c->capacity()) : -1;
}

int32_t sr_score_cache_get(sr_score_cache* c, const char* searcher_id, uint64_t query_signature,
                           int64_t entity_id, const char* model_version, double* scores,
                           int32_t n_tasks, int32_t* hit) {
  return guard([&] {
    if (!c || !searcher_id || !model_version || !scores || !hit)
      srh::fail(SR_SPEC_VIOLATION, "null argument");
    *hit = c->c->get({searcher_id, query_signature, entity_id, model_version}, scores, n_tasks) ? 1 : 0;
  });
}

int32_t sr_score_cache_put(sr_score_cache* c, const char* searcher_id, uint64_t query_signature,
                           int64_t entity_id, const char* model_version, const double* scores,
                           int32_t n_tasks) {
  return guard([&] {
    if (!c || !searcher_id || !model_version || !scores)
      srh::fail(SR_SPEC_VIOLATION, "null argument");
    if (n_tasks < 1) srh::fail(SR_PARAMETER, "n_tasks must be >= 1");
    c->c->put({searcher_id, query_signature, entity_id, model_version}, scores, n_tasks);
  });
}

namespace {
std::string canonical_of(const char* text, int32_t n_filters, const char* const* attrs,
                         const char* const* values) {
  if (!text || n_filters < 0 || (n_filters > 0 && (!attrs || !values)))
    srh::fail(SR_SPEC_VIOLATION, "null argument");
  std::vector<std::pair<std::string, std::string>> f;
  f.reserve(static_cast<size_t>(n_filters));
  for (int32_t i = 0; i < n_filters; ++i) {
    if (!attrs[i] || !values[i]) srh::fail(SR_SPEC_VIOLATION, "null filter string");
    f.emplace_back(attrs[i], values[i]);
  }
  return srh::canonical_query(text, f);
}
}  // namespace

int32_t sr_canonical_query(const char* text, int32_t n_filters, const char* const* attrs,
                           const char* const* values, char* out, int64_t cap, int64_t* len) {
  return guard([&] {
    if (!len) srh::fail(SR_SPEC_VIOLATION, "null argument");
    const std::string s = canonical_of(text, n_filters, attrs, values);
    if (out && cap > 0) std::memcpy(out, s.data(), std::min<size_t>(s.size(), static_cast<size_t>(cap)));
    *len = static_cast<int64_t>(s.size());
  });
}

int32_t sr_query_signature(const char* text, int32_t n_filters, const char* const* attrs,
                           const char* const* values, uint64_t* out) {
  return guard([&] {
    if (!out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    *out = srh::fnv1a64(canonical_of(text, n_filters, attrs, values));
  });
}

uint64_t sr_fnv1a64(const char* data, int64_t len) {
  return srh::fnv1a64(data ? data : "", data && len > 0 ? static_cast<size_t>(len) : 0);
}

int32_t sr_engine_score_cached(sr_engine* e, sr_score_cache* c, const char* searcher_id,
                               uint64_t query_signature, const char* model_version,
                               const sr_request* req, sr_result* res, int32_t* n_hits) {
  return guard([&] {
    if (!e || !c || !searcher_id || !model_version || !req || !res)
      srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    e->e->score_cached(*c->c, searcher_id, query_signature, model_version, *req, res, n_hits);
  });
}

int32_t sr_engine_reserve(sr_engine* e, int64_t rows) {
  return guard([&] {
    if (!e) srh::fail(SR_SPEC_VIOLATION, "null argument");
    if (rows < 1 || rows > (int64_t(1) << 29)) srh::fail(SR_PARAMETER, "reserve rows must be in [1, 2^29]");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    e->e->reserve(static_cast<int32_t>(rows));
  });
}

int32_t sr_engine_set_projection(sr_engine* e, const float* proj, int32_t d_emb, int32_t n_soft) {
  return guard([&] {
    if (!e) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    e->e->set_projection(proj, d_emb, n_soft);
  });
}

int32_t sr_engine_score_emb(sr_engine* e, const int32_t* prefix, int32_t t_q, const float* emb,
                            int32_t d_emb, int32_t n_items, const int64_t* item_ids,
                            int32_t form, sr_result* res) {
  return guard([&] {
    if (!e || !res || (t_q > 0 && !prefix)) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    e->e->score_emb(prefix, t_q, emb, d_emb, n_items, item_ids, form, res);
  });
}

int32_t sr_plan_create_emb(sr_engine* e, const int32_t* prefix, int32_t t_q, const float* emb,
                           int32_t d_emb, int32_t n_items, const int64_t* item_ids, int32_t form,
                           int32_t k, sr_plan** out) {
  return guard([&] {
    if (!e || !out || (t_q > 0 && !prefix)) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    auto p = std::make_unique<sr_plan>();
    p->owner = e;
    p->p = e->e->make_plan_emb(prefix, t_q, emb, d_emb, n_items, item_ids, form, k);
    *out = p.release();
  });
}

int32_t sr_engine_device(const sr_engine* e) { return e ? e->e->device() : -1; }
void* sr_engine_stream(const sr_engine* e) { return e ? e->e->stream() : nullptr; }

int32_t sr_plan_create(sr_engine* e, const sr_request* req, int32_t k, sr_plan** out) {
  return guard([&] {
    if (!e || !req || !out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    auto p = std::make_unique<sr_plan>();
    p->owner = e;
    p->p = e->e->make_plan(req, 1, k);
    *out = p.release();
  });
}

int32_t sr_plan_create_batch(sr_engine* e, const sr_request* reqs, int32_t n_req, int32_t k,
                             sr_plan** out) {
  return guard([&] {
    if (!e || !reqs || !out || n_req <= 0) srh::fail(SR_SPEC_VIOLATION, "bad argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    auto p = std::make_unique<sr_plan>();
    p->owner = e;
    p->p = e->e->make_plan(reqs, n_req, k);
    *out = p.release();
  });
}

int32_t sr_plan_fetch_batch(sr_plan* p, sr_result* res, int32_t n_req) {
  return guard([&] {
    if (!p || !res) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(p->owner->e->mutex());
    if (n_req != static_cast<int32_t>(p->p->reqs.size()))
      srh::fail(SR_PARAMETER, "result count differs from the plan's request count");
    p->owner->e->fetch(*p->p, res, n_req);
  });
}

int32_t sr_plan_run(sr_plan* p) {
  return guard([&] {
    if (!p) srh::fail(SR_SPEC_VIOLATION, "null plan");
    std::lock_guard<std::mutex> lock(p->owner->e->mutex());
    p->owner->e->run_plan(*p->p);
    p->sharded_valid = false;
  });
}

int32_t sr_plan_sync(sr_plan* p) {
  return guard([&] {
    if (!p) srh::fail(SR_SPEC_VIOLATION, "null plan");
    std::lock_guard<std::mutex> lock(p->owner->e->mutex());
    SR_CUDA_CHECK(cudaStreamSynchronize(p->owner->e->stream()));
  });
}

int32_t sr_plan_fetch(sr_plan* p, sr_result* res) {
  return guard([&] {
    if (!p || !res) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(p->owner->e->mutex());
    p->owner->e->fetch(*p->p, res, 1);
    if (p->sharded_valid) copy_topk_merged(*p->p, res, p->owner->e->stream());
  });
}

int32_t sr_plan_kernel_count(const sr_plan* p, int32_t* launches) {
  return guard([&] {
    if (!p || !launches) srh::fail(SR_SPEC_VIOLATION, "null argument");
    *launches = p->p->launches;
  });
}

int32_t sr_plan_profile(sr_plan* p, int32_t reps, float* ms_out, int32_t* launches_out) {
  return guard([&] {
    if (!p) srh::fail(SR_SPEC_VIOLATION, "null plan");
    std::lock_guard<std::mutex> lock(p->owner->e->mutex());
    p->owner->e->profile(*p->p, reps, ms_out, launches_out);
  });
}

int32_t sr_plan_shape(const sr_plan* p, int64_t* out8) {
  return guard([&] {
    if (!p || !out8) srh::fail(SR_SPEC_VIOLATION, "null argument");
    const auto& pk = p->p->pack;
    out8[0] = pk.M;
    out8[1] = pk.n_items;
    out8[2] = static_cast<int64_t>(pk.tiles.size());
    out8[3] = pk.n_soft;
    int64_t h2d = 0;
    h2d += static_cast<int64_t>(pk.row_src.size()) * 4 + static_cast<int64_t>(pk.row_pos.size()) * 4;
    h2d += static_cast<int64_t>(pk.spans.size()) * sizeof(srk::RowSpan);
    h2d += static_cast<int64_t>(pk.tiles.size()) * sizeof(srk::AttnTile);
    h2d += static_cast<int64_t>(pk.last_rows.size()) * 4 + static_cast<int64_t>(pk.ids.size()) * 8;
    h2d += static_cast<int64_t>(pk.seg_off.size()) * 4;
    if (p->p->emb_form >= 0)  // compact embeddings; the rows are made on the device
      h2d += static_cast<int64_t>(p->p->emb_n) * p->p->emb_d * 4;
    else
      h2d += static_cast<int64_t>(pk.n_soft) * 4 * p->owner->e->config().d_model;
    out8[4] = h2d;
    out8[5] = static_cast<int64_t>(pk.n_items) * p->p->n_tasks * 8 +
              static_cast<int64_t>(pk.seg_off.size() - 1) * p->p->k * sizeof(srk::TopkEntry);
    out8[6] = p->p->k;
    out8[7] = p->p->n_tasks;
  });
}

void sr_plan_destroy(sr_plan* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lock(p->owner->e->mutex());  // graph/buffers freed off the stream
  delete p;
}

int32_t sr_nccl_unique_id(uint8_t out[128]) {
  return guard([&] { srh::nccl_unique_id(out); });
}

int32_t sr_comm_create(int32_t nranks, int32_t rank, const uint8_t id[128], int32_t device,
                       sr_comm** out) {
  return guard([&] {
    auto c = std::make_unique<sr_comm>();
    c->c = srh::comm_create(nranks, rank, id, device);
    *out = c.release();
  });
}

int32_t sr_comm_create_host(int32_t nranks, int32_t rank, int32_t device, sr_allgather_fn fn,
                            void* user, sr_comm** out) {
  return guard([&] {
    if (!out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    auto c = std::make_unique<sr_comm>();
    c->c = srh::comm_create_host(nranks, rank, device, fn, user);
    *out = c.release();
  });
}

void sr_comm_destroy(sr_comm* c) {
  if (c) srh::comm_destroy(c->c);
  delete c;
}

int32_t sr_engine_score_sharded(sr_engine* e, sr_comm* c, const sr_request* local_shard,
                                sr_result* res) {
  return guard([&] {
    if (!e || !c || !local_shard || !res) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(e->e->mutex());
    auto p = e->e->make_plan(local_shard, 1, res->k);
    e->e->run_plan_sharded(*p, c->c);
    e->e->fetch(*p, res, 1);
    copy_topk_merged(*p, res, e->e->stream());
  });
}

int32_t sr_plan_run_sharded(sr_plan* p, sr_comm* c) {
  return guard([&] {
    if (!p || !c) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(p->owner->e->mutex());
    p->owner->e->run_plan_sharded(*p->p, c->c);
    p->sharded_valid = true;
  });
}

// ------------------------------------------------------------ retrieval
int32_t sr_corpus_create(const float* embeddings, const float* features, const int64_t* doc_ids,
                         int64_t n_docs, int32_t d_emb, int32_t n_features, int32_t device,
                         sr_corpus** out) {
  return guard([&] {
    if (!out) srh::fail(SR_SPEC_VIOLATION, "null argument");
    if (n_docs > 0 && (!embeddings || !doc_ids || (n_features > 0 && !features)))
      srh::fail(SR_SPEC_VIOLATION, "null corpus array");
    auto c = std::make_unique<sr_corpus>();
    c->c = std::make_unique<srh::Corpus>(embeddings, features, doc_ids, n_docs, d_emb, n_features,
                                         device);
    *out = c.release();
  });
}

void sr_corpus_destroy(sr_corpus* c) { delete c; }

int32_t sr_corpus_topk(sr_corpus* c, const float* query, int32_t d_query, double w0,
                       const double* w, int32_t n_w, const uint8_t* keep, int32_t k,
                       int64_t* ids_out, double* scores_out, int32_t* n_out) {
  return guard([&] {
    if (!c || !query || !n_out || (n_w > 0 && !w)) srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(c->mu);
    *n_out = c->c->topk_host(query, d_query, w0, w, n_w, keep, k, ids_out, scores_out);
  });
}

int32_t sr_corpus_topk_sharded(sr_corpus* c, sr_comm* comm, const float* query, int32_t d_query,
                               double w0, const double* w, int32_t n_w, const uint8_t* keep,
                               int32_t k, int64_t* ids_out, double* scores_out, int32_t* n_out) {
  return guard([&] {
    if (!c || !comm || !query || !n_out || (n_w > 0 && !w))
      srh::fail(SR_SPEC_VIOLATION, "null argument");
    std::lock_guard<std::mutex> lock(c->mu);
    *n_out = c->c->topk_sharded(comm->c, query, d_query, w0, w, n_w, keep, k, ids_out, scores_out);
  });
}

int64_t sr_corpus_last_candidates(const sr_corpus* c) {
  return c ? c->c->last_candidates() : 0;
}

float sr_corpus_last_scan_ms(const sr_corpus* c) { return c ? c->c->last_scan_ms() : 0.f; }

// ------------------------------------------------------------ kernel tests
int32_t sr_kernel_gemm(const void* a_bf16, const void* b_bf16, int32_t M, int32_t N, int32_t K,
                       void* c, int32_t ldc, int32_t epi, void* stream) {
  return guard([&] {
    const int bn = srk::gemm_pick_bn(N);
    if (bn == 0) srh::fail(SR_SPEC_VIOLATION, "N must be a multiple of 64");
    if (K % 8 != 0) srh::fail(SR_SPEC_VIOLATION, "K must be a multiple of 8");
    CUtensorMap ta, tb;
    SR_CUDA_CHECK(srk::make_tmap_bf16_2d(&ta, a_bf16, M, K, 128, 64));
    SR_CUDA_CHECK(srk::make_tmap_bf16_2d(&tb, b_bf16, N, K, srk::gemm_b_box_rows(N), 64));
    SR_CUDA_CHECK(srk::gemm_auto(ta, tb, M, N, K, c, ldc, epi, static_cast<cudaStream_t>(stream)));
    // NULL stream: synchronous (errors surface here); explicit stream: async.
    if (stream == nullptr) SR_CUDA_CHECK(cudaStreamSynchronize(nullptr));
  });
}

int32_t sr_kernel_gemm_resid_ln(const void* a_bf16, const void* b_bf16, int32_t M, int32_t N,
                                int32_t K, float* x, const float* gain, void* out_bf16,
                                uint32_t* counters, void* stream) {
  return guard([&] {
    if (!srk::gemm_use_pair(N) || N > 2048) srh::fail(SR_SPEC_VIOLATION, "N must be a multiple of 256, <= 2048");
    if (K % 8 != 0) srh::fail(SR_SPEC_VIOLATION, "K must be a multiple of 8");
    if (!x || !gain || !out_bf16 || !counters) srh::fail(SR_SPEC_VIOLATION, "null argument");
    CUtensorMap ta, tb;
    SR_CUDA_CHECK(srk::make_tmap_bf16_2d(&ta, a_bf16, M, K, 128, 64));
    SR_CUDA_CHECK(srk::make_tmap_bf16_2d(&tb, b_bf16, N, K, srk::gemm_b_box_rows(N), 64));
    srk::LnFold f{};
    f.ln_cnt = counters;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // side stream + fork/join events, released on every path (RAII)
    struct Side {
      cudaStream_t s2 = nullptr;
      cudaEvent_t fork = nullptr, join = nullptr;
      ~Side() {
        if (fork) cudaEventDestroy(fork);
        if (join) cudaEventDestroy(join);
        if (s2) cudaStreamDestroy(s2);
      }
    } sd;
    SR_CUDA_CHECK(cudaStreamCreateWithFlags(&sd.s2, cudaStreamNonBlocking));
    SR_CUDA_CHECK(cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming));
    SR_CUDA_CHECK(cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming));
    SR_CUDA_CHECK(cudaEventRecord(sd.fork, s));
    SR_CUDA_CHECK(cudaStreamWaitEvent(sd.s2, sd.fork, 0));
    SR_CUDA_CHECK(srk::gemm_auto(ta, tb, M, N, K, x, N, srk::EPI_RESID_F32_LN, s, &f));
    SR_CUDA_CHECK(srk::layer_norm_after(x, gain, static_cast<__nv_bfloat16*>(out_bf16), M, N,
                                        counters, N / 256, sd.s2));
    SR_CUDA_CHECK(cudaEventRecord(sd.join, sd.s2));
    SR_CUDA_CHECK(cudaStreamWaitEvent(s, sd.join, 0));
    SR_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int32_t sr_kernel_gemm_ln(const void* a_bf16, const void* b_bf16, int32_t M, int32_t N, int32_t K,
                          void* c, int32_t ldc, int32_t epi, void* xb_bf16, void* stats,
                          int32_t n_parts, const float* colsum, int32_t ld, void* stream) {
  return guard([&] {
    if (epi < srk::EPI_RESID_LN || epi > srk::EPI_LN_GELU_BF16)
      srh::fail(SR_PARAMETER, "epi must be 4, 5 or 6");
    if (!srk::gemm_use_pair(N)) srh::fail(SR_SPEC_VIOLATION, "N must be a multiple of 256");
    if (K % 8 != 0) srh::fail(SR_SPEC_VIOLATION, "K must be a multiple of 8");
    CUtensorMap ta, tb;
    SR_CUDA_CHECK(srk::make_tmap_bf16_2d(&ta, a_bf16, M, K, 128, 64));
    SR_CUDA_CHECK(srk::make_tmap_bf16_2d(&tb, b_bf16, N, K, srk::gemm_b_box_rows(N), 64));
    srk::LnFold f{};
    f.ld = ld;
    if (epi == srk::EPI_RESID_LN) {
      f.xb = static_cast<__nv_bfloat16*>(xb_bf16);
      f.stats_out = static_cast<float*>(stats);
    } else {
      f.stats_in = static_cast<const float*>(stats);
      f.colsum = colsum;
      f.n_parts = n_parts;
    }
    SR_CUDA_CHECK(srk::gemm_auto(ta, tb, M, N, K, c, ldc, epi, static_cast<cudaStream_t>(stream), &f));
    if (stream == nullptr) SR_CUDA_CHECK(cudaStreamSynchronize(nullptr));
  });
}

int32_t sr_kernel_attention(const void* qkv, const int32_t* spans_host, int32_t M,
                            int32_t n_heads, int32_t head_dim, void* out, void* stream) {
  return guard([&] {
    // Tiles: 64-row query tiles; keys = [min prefix_begin, max prefix_end) and
    // [min span_start, q_end) (ranges merged when they touch).
    std::vector<srk::RowSpan> spans(M);
    std::memcpy(spans.data(), spans_host, sizeof(srk::RowSpan) * M);
    std::vector<srk::AttnTile> tiles;
    const int tr = srk::attention_tile_rows(head_dim);
    for (int r0 = 0; r0 < M; r0 += tr) {
      const int r1 = std::min(M, r0 + tr);
      int pb = INT32_MAX, pe = 0, ss = INT32_MAX;
      for (int r = r0; r < r1; ++r) {
        const auto& s = spans[r];
        if (s.prefix_begin < 0 || s.prefix_end < s.prefix_begin || s.span_start < s.prefix_end ||
            s.span_start > r)
          srh::fail(SR_MASK_INVALID, "mask entry " + std::to_string(r) +
                                         " violates prefix_end <= span_start <= position");
        if (s.prefix_end > s.prefix_begin) {
          pb = std::min(pb, s.prefix_begin);
          pe = std::max(pe, s.prefix_end);
        }
        ss = std::min(ss, s.span_start);
      }
      srk::AttnTile t{r0, r1, 0, 0, ss, r1, 0, 0};
      if (pe > 0) {
        if (pe >= ss) {  // overlapping ranges: one contiguous range
          t.r2_begin = std::min(pb, ss);
        } else {
          t.r1_begin = pb;
          t.r1_end = pe;
        }
      }
      tiles.push_back(t);
    }
    srk::RowSpan* dsp = nullptr;
    srk::AttnTile* dt = nullptr;
    SR_CUDA_CHECK(cudaMalloc(&dsp, sizeof(srk::RowSpan) * M));
    SR_CUDA_CHECK(cudaMalloc(&dt, sizeof(srk::AttnTile) * tiles.size()));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaMemcpy(dsp, spans.data(), sizeof(srk::RowSpan) * M, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, tiles.data(), sizeof(srk::AttnTile) * tiles.size(), cudaMemcpyHostToDevice);
    cudaError_t err;
    int2* dw = nullptr;
    if (head_dim >= 64) {
      CUtensorMap tm;
      err = srk::make_tmap_bf16_2d(&tm, qkv, M, 3 * n_heads * head_dim, 128, 64);
      // the engine's LPT work order (SRK_ATTN_LPT=0: head-major)
      std::vector<int2> work;
      const char* lpt = std::getenv("SRK_ATTN_LPT");
      if (lpt == nullptr || std::atoi(lpt) != 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        srk::attention_work_lpt(tiles.data(), static_cast<int>(tiles.size()), n_heads,
                                srk::attention_ctas(static_cast<int>(tiles.size()), n_heads, dev),
                                work);
        if (err == cudaSuccess) err = cudaMalloc(&dw, sizeof(int2) * work.size());
        if (err == cudaSuccess)
          err = cudaMemcpy(dw, work.data(), sizeof(int2) * work.size(), cudaMemcpyHostToDevice);
      }
      if (err == cudaSuccess)
        err = srk::attention_tc(tm, qkv, dsp, dt, static_cast<int>(tiles.size()),
                                static_cast<__nv_bfloat16*>(out), M, n_heads, head_dim, s, dw,
                                static_cast<int>(work.size()));
    } else {
      err = srk::attention(static_cast<const __nv_bfloat16*>(qkv), dsp, dt,
                           static_cast<int>(tiles.size()), static_cast<__nv_bfloat16*>(out), M,
                           n_heads, head_dim, s);
    }
    if (err == cudaSuccess) err = cudaStreamSynchronize(s);
    cudaFree(dsp);
    cudaFree(dt);
    if (dw) cudaFree(dw);
    SR_CUDA_CHECK(err);
  });
}

int32_t sr_kernel_layernorm(const float* x, const float* gain, void* out_bf16, int32_t M,
                            int32_t d, void* stream) {
  return guard([&] {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    SR_CUDA_CHECK(srk::layer_norm_bf16(x, gain, static_cast<__nv_bfloat16*>(out_bf16), M, d, s));
    SR_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

int32_t sr_debug_attention_trace(void* dev_buf) {
  return guard([&] {
    SR_CUDA_CHECK(srk::attention_set_trace(static_cast<unsigned long long*>(dev_buf)));
  });
}

int32_t sr_debug_gemm_trace(void* dev_buf) {
  return guard([&] { SR_CUDA_CHECK(srk::gemm_set_trace(static_cast<unsigned long long*>(dev_buf))); });
}

int32_t sr_kernel_topk(const double* scores, const int64_t* ids, int32_t n, int32_t k,
                       int64_t* ids_out_host, double* scores_out_host, int32_t* index_out_host) {
  return guard([&] {
    if (n <= 0 || k <= 0) srh::fail(SR_PARAMETER, "n and k must be >= 1");
    int32_t* seg = nullptr;
    srk::TopkEntry *scratch = nullptr, *out = nullptr;
    const int chunks = (n + 4095) / 4096;
    const int32_t off[2] = {0, n};
    SR_CUDA_CHECK(cudaMalloc(&seg, sizeof(off)));
    SR_CUDA_CHECK(cudaMalloc(&scratch, sizeof(srk::TopkEntry) * chunks * k));
    SR_CUDA_CHECK(cudaMalloc(&out, sizeof(srk::TopkEntry) * k));
    cudaMemcpy(seg, off, sizeof(off), cudaMemcpyHostToDevice);
    cudaError_t err =
        srk::topk(scores, 1, ids, seg, 1, n, k, scratch, chunks * k, out, nullptr);
    std::vector<srk::TopkEntry> h(k);
    if (err == cudaSuccess)
      err = cudaMemcpy(h.data(), out, sizeof(srk::TopkEntry) * k, cudaMemcpyDeviceToHost);
    cudaFree(seg);
    cudaFree(scratch);
    cudaFree(out);
    SR_CUDA_CHECK(err);
    for (int j = 0; j < std::min(k, n); ++j) {
      if (ids_out_host) ids_out_host[j] = h[j].id;
      if (scores_out_host) scores_out_host[j] = h[j].score;
      if (index_out_host) index_out_host[j] = h[j].index;
    }
  });
}

}  // extern "C"
