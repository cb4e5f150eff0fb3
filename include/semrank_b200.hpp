// semrank_b200.hpp — header-only C++ facade over the C-ABI with the
// reference's own type names (namespace semrank; engine.hpp / model.hpp /
// weights_io.hpp / error.hpp), so a caller such as the reference's
// service.cpp (service.cpp:224 `engine_.score(score_request)`) relinks against
// libsemrank_b200.so instead of the CPU scorer. Differences from the
// reference API, all additive:
//   * ModelWeights is an owning handle (weights live in the library);
//   * ScoringEngine takes a device index and owns device copies;
//   * ScoringEngine::score takes an optional top-k length and fills
//     ScoreResult::topk (caller-side ordering, semrank_main.cpp:393-398).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "semrank_b200.h"

namespace semrank {

enum class ErrorCode {  // error.hpp:13-29 (same order)
  LengthOverflow, MaskInvalid, SpecViolation, PayloadInvalid, SchemaUnknown, Alignment,
  Divergence, Parameter, DegenerateInput, UndefinedMetric, StateInvalid, OversizeItem,
  Consistency, Reconciliation, Io
};

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& m) : std::runtime_error(m), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

// Device-side failures (CUDA / NCCL) have no reference equivalent.
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(int32_t st) {
  if (st == SR_OK) return;
  const std::string msg = sr_last_error();
  if (st >= 1 && st <= 15) throw Error(static_cast<ErrorCode>(st - 1), msg);
  throw DeviceError(std::string(sr_status_name(st)) + ": " + msg);
}

enum class ScoreMode { Naive, Ibpc, MultiItem, Mixed };  // engine.hpp:15

struct HeadSpec {
  std::string name;
  int arity = 1;
};

struct ModelConfig {  // model.hpp:24-40
  int n_layers = 2, d_model = 64, n_heads = 4, d_ff = 256, vocab_size = 300, max_seq = 4096;
  int yes_token_id = 261, no_token_id = 262;
  std::vector<HeadSpec> head_specs;
  int head_dim() const { return d_model / n_heads; }
  static ModelConfig default_toy() {
    ModelConfig c;
    c.head_specs = {{"click", 1}, {"apply", 1}, {"badfit", 1}, {"shortlist", 1}, {"dismiss", 1}};
    return c;
  }
  void validate() const { with_c([](const sr_model_config& c) { check(sr_config_validate(&c)); }); }

  template <typename F>
  void with_c(F&& f) const {
    std::vector<const char*> names;
    std::vector<int32_t> ar;
    for (const auto& h : head_specs) {
      names.push_back(h.name.c_str());
      ar.push_back(h.arity);
    }
    sr_model_config c{n_layers, d_model, n_heads, d_ff, vocab_size, max_seq, yes_token_id,
                      no_token_id, static_cast<int32_t>(head_specs.size()), names.data(),
                      ar.data()};
    f(c);
  }
};

class ModelWeights {  // model.hpp:56-67, owning handle
 public:
  explicit ModelWeights(sr_weights* w) : w_(w, &sr_weights_free) {
    sr_model_config c{};
    check(sr_weights_config(w, &c));
    config.n_layers = c.n_layers;
    config.d_model = c.d_model;
    config.n_heads = c.n_heads;
    config.d_ff = c.d_ff;
    config.vocab_size = c.vocab_size;
    config.max_seq = c.max_seq;
    config.yes_token_id = c.yes_token_id;
    config.no_token_id = c.no_token_id;
    for (int i = 0; i < c.n_task_heads; ++i)
      config.head_specs.push_back({c.head_names[i], c.head_arity[i]});
    version = sr_weights_version(w);
    for (size_t i = 0; i < sr_weights_tensor_count(w); ++i) {
      const char* name = nullptr;
      float* data = nullptr;
      size_t numel = 0;
      check(sr_weights_tensor(w, i, &name, &data, &numel));
      if (std::string(name) == "tok_emb") tok_emb = TensorView{data, numel};
      if (std::string(name) == "pos_emb") pos_emb = TensorView{data, numel};
    }
  }
  // Read-only views of the embedding tables (model.hpp:58-59: tok_emb
  // [V x d], pos_emb [max_seq x d]); valid while any copy of the handle lives.
  struct TensorView {
    const float* p = nullptr;
    size_t n = 0;
    const float* data() const { return p; }
    size_t size() const { return n; }
    float operator[](size_t i) const { return p[i]; }
  };
  ModelConfig config;
  std::string version;
  TensorView tok_emb, pos_emb;
  const sr_weights* handle() const { return w_.get(); }

 private:
  std::shared_ptr<sr_weights> w_;
};

inline ModelWeights init_model(const ModelConfig& cfg, std::uint64_t seed,
                               sr_init_scheme scheme = SR_INIT_REFERENCE) {  // model.cpp:94-134
  sr_weights* w = nullptr;
  cfg.with_c([&](const sr_model_config& c) { check(sr_weights_init(&c, seed, scheme, &w)); });
  return ModelWeights(w);
}
inline ModelWeights load_weights(const std::string& path) {  // weights_io.cpp:137-196
  sr_weights* w = nullptr;
  check(sr_weights_load(path.c_str(), &w));
  return ModelWeights(w);
}
inline void save_weights(const ModelWeights& w, const std::string& path) {
  check(sr_weights_save(w.handle(), path.c_str()));
}

struct ScoreItem {  // engine.hpp:20-25
  std::string id;
  std::vector<int> tokens;
  std::vector<float> embedding;  // mixed: [n_emb_tokens x d_model]
  int n_emb_tokens = 0;
};

struct ScoreRequest {  // engine.hpp:27-33
  std::string request_id;
  std::vector<int> prefix_tokens;
  std::vector<ScoreItem> items;
  ScoreMode mode = ScoreMode::Ibpc;
  bool latency_sensitive = false;
};

struct FlopReport {  // engine.hpp:38-44
  double attention_units = 0, linear_units = 0, t_q = 0, t_i_mean = 0, n_items = 0;
};

inline FlopReport flops(ScoreMode mode, long t_q, long t_i, long n_items) {  // engine.cpp:30-47
  sr_flop_report r{};
  check(sr_flops(static_cast<int32_t>(mode), t_q, t_i, n_items, &r));
  return {r.attention_units, r.linear_units, r.t_q, r.t_i_mean, r.n_items};
}

struct ItemScores {  // engine.hpp:46-49
  std::string item_id;
  std::map<std::string, double> tasks;
};

struct ScoreResult {  // engine.hpp:53-59 (+ topk)
  std::string request_id;
  std::vector<ItemScores> items;
  ScoreMode mode = ScoreMode::Naive;
  FlopReport flops;
  double kv_incremental_per_item = 0;
  std::vector<std::pair<std::string, double>> topk;  // (item id, relevance), best first
};

inline constexpr const char* kRelevanceTask = "relevance";

// ----------------------------------------------- mid-tier score cache
// midtier.hpp:16-69 over sr_score_cache / sr_canonical_query / sr_fnv1a64.
inline std::string canonical_query(const std::string& query_text,
                                   const std::map<std::string, std::vector<std::string>>& filters) {
  std::vector<const char*> attrs, values;
  for (const auto& [attr, vs] : filters)
    for (const auto& v : vs) {
      attrs.push_back(attr.c_str());
      values.push_back(v.c_str());
    }
  int64_t len = 0;
  const int32_t n = static_cast<int32_t>(attrs.size());
  check(sr_canonical_query(query_text.c_str(), n, attrs.data(), values.data(), nullptr, 0, &len));
  std::string out(static_cast<size_t>(len), '\0');
  check(sr_canonical_query(query_text.c_str(), n, attrs.data(), values.data(), out.data(), len,
                           &len));
  return out;
}

inline std::uint64_t fnv1a64(const std::string& text) {
  return sr_fnv1a64(text.data(), static_cast<int64_t>(text.size()));
}

struct CacheKey {  // midtier.hpp:30-37
  std::string searcher_id;
  std::uint64_t query_signature = 0;
  std::int64_t entity_id = 0;
  std::string model_version;
  bool operator==(const CacheKey& o) const {
    return searcher_id == o.searcher_id && query_signature == o.query_signature &&
           entity_id == o.entity_id && model_version == o.model_version;
  }
};

using TaskScoreMap = std::map<std::string, double>;

class ScoreCache {  // midtier.hpp:42-69; rows kept in task order
 public:
  explicit ScoreCache(std::size_t capacity)
      : ScoreCache(capacity, default_tasks()) {}
  ScoreCache(std::size_t capacity, std::vector<std::string> task_names)
      : tasks_(std::move(task_names)) {
    sr_score_cache* c = nullptr;
    check(sr_score_cache_create(static_cast<int64_t>(capacity), &c));
    c_.reset(c);
  }
  std::optional<TaskScoreMap> get(const CacheKey& key) {
    std::vector<double> row(tasks_.size());
    int32_t hit = 0;
    check(sr_score_cache_get(c_.get(), key.searcher_id.c_str(), key.query_signature, key.entity_id,
                             key.model_version.c_str(), row.data(),
                             static_cast<int32_t>(row.size()), &hit));
    if (!hit) return std::nullopt;
    TaskScoreMap m;
    for (size_t i = 0; i < tasks_.size(); ++i) m[tasks_[i]] = row[i];
    return m;
  }
  void put(const CacheKey& key, const TaskScoreMap& scores) {
    std::vector<double> row;
    for (const auto& t : tasks_) {
      const auto it = scores.find(t);
      if (it == scores.end() || scores.size() != tasks_.size())
        throw Error(ErrorCode::Alignment, "score map does not match the cache's tasks");
      row.push_back(it->second);
    }
    check(sr_score_cache_put(c_.get(), key.searcher_id.c_str(), key.query_signature, key.entity_id,
                             key.model_version.c_str(), row.data(),
                             static_cast<int32_t>(row.size())));
  }
  std::size_t size() const { return static_cast<std::size_t>(sr_score_cache_size(c_.get())); }
  std::size_t capacity() const {
    return static_cast<std::size_t>(sr_score_cache_capacity(c_.get()));
  }
  sr_score_cache* handle() const { return c_.get(); }

 private:
  static std::vector<std::string> default_tasks() {
    std::vector<std::string> t{kRelevanceTask};
    for (const auto& h : ModelConfig::default_toy().head_specs) t.push_back(h.name);
    return t;
  }
  struct Del {
    void operator()(sr_score_cache* c) const { sr_score_cache_destroy(c); }
  };
  std::vector<std::string> tasks_;
  std::unique_ptr<sr_score_cache, Del> c_;
};

// Exhaustive retrieval top-K on the device: replaces
// exhaustive_topk (retrieval.hpp:60-70, retrieval.cpp:134-173) — score =
// w0 cos(q, e_d) + sum_i w_i f_i(d), exact top-K by (score desc, doc_id asc),
// scores identical to the reference's doubles. The corpus is columnar and
// copied to the device once; filters are the caller's keep mask
// (filter_candidates, retrieval.cpp:79-97).
struct RankedDoc {  // retrieval.hpp:59-62
  std::int64_t doc_id = 0;
  double score = 0;
  bool operator==(const RankedDoc& o) const { return doc_id == o.doc_id && score == o.score; }
};
class Corpus {
 public:
  Corpus(const std::vector<float>& embeddings, const std::vector<float>& features,
         const std::vector<std::int64_t>& doc_ids, int d_emb, int n_features, int device = 0) {
    const std::int64_t n = static_cast<std::int64_t>(doc_ids.size());
    if (embeddings.size() != static_cast<size_t>(n) * d_emb ||
        features.size() != static_cast<size_t>(n) * n_features)
      throw Error(ErrorCode::Alignment, "corpus columns do not match the document count");
    sr_corpus* c = nullptr;
    check(sr_corpus_create(embeddings.data(), features.empty() ? nullptr : features.data(),
                           doc_ids.data(), n, d_emb, n_features, device, &c));
    c_.reset(c);
  }
  std::vector<RankedDoc> topk(const std::vector<float>& query, double w0,
                              const std::vector<double>& w, int k,
                              const std::vector<std::uint8_t>& keep = {}) {
    std::vector<std::int64_t> ids(k > 0 ? k : 1);
    std::vector<double> sc(k > 0 ? k : 1);
    int32_t n = 0;
    check(sr_corpus_topk(c_.get(), query.data(), static_cast<int32_t>(query.size()), w0,
                         w.empty() ? nullptr : w.data(), static_cast<int32_t>(w.size()),
                         keep.empty() ? nullptr : keep.data(), k, ids.data(), sc.data(), &n));
    std::vector<RankedDoc> out;
    for (int i = 0; i < n; ++i) out.push_back({ids[i], sc[i]});
    return out;
  }

 private:
  struct Del {
    void operator()(sr_corpus* c) const { sr_corpus_destroy(c); }
  };
  std::unique_ptr<sr_corpus, Del> c_;
};

class Scheduler;

// Candidate sharding across GPUs: one process per GPU, each
// scoring a contiguous shard of the items with global item ids; the per-rank
// top-k lists are merged with the reference's comparator
// (retrieval.cpp:144-165) over NCCL. Rank 0 makes the id, the caller's own
// bootstrap broadcasts it, every rank constructs a Comm.
class Comm {
 public:
  using Id = std::vector<std::uint8_t>;
  static Id unique_id() {
    Id id(128);
    check(sr_nccl_unique_id(id.data()));
    return id;
  }
  Comm(int nranks, int rank, const Id& id, int device) {
    if (id.size() != 128) throw Error(ErrorCode::Parameter, "NCCL id must be 128 bytes");
    sr_comm* c = nullptr;
    check(sr_comm_create(nranks, rank, id.data(), device, &c));
    c_.reset(c);
  }
  sr_comm* handle() const { return c_.get(); }

 private:
  struct Del {
    void operator()(sr_comm* c) const { sr_comm_destroy(c); }
  };
  std::unique_ptr<sr_comm, Del> c_;
};

class ScoringEngine {  // engine.hpp:109-119
 public:
  explicit ScoringEngine(const ModelWeights& weights, int device = 0) : weights_(weights) {
    if (sr_abi_version() != SR_ABI_VERSION)  // header and library built apart
      throw Error(ErrorCode::StateInvalid, "libsemrank_b200 C-ABI version differs from the header's");
    sr_engine* e = nullptr;
    check(sr_engine_create(weights.handle(), device, &e));
    e_.reset(e);
  }
  const ModelWeights& weights() const { return weights_; }

  ScoreResult score(const ScoreRequest& request, int k = 0) {
    return score_as(request, request.mode, k);
  }

  // Scores `request` as if request.mode were `mode` (the free score_naive /
  // score_ibpc / ... functions of engine.hpp:77-86).
  ScoreResult score_as(const ScoreRequest& request, ScoreMode mode, int k = 0) {
    Packed p(request, weights_.config.d_model, mode);
    Out o(request.items.size(), 1 + weights_.config.head_specs.size(), k);
    check(sr_engine_score(e_.get(), &p.req, &o.res));
    auto r = o.result(request, weights_.config);
    r.mode = mode;
    return r;
  }

  // Several requests in one packed device pass (plan_batches generalised,
  // engine.cpp:278-326); results in request order.
  std::vector<ScoreResult> score_batch(const std::vector<ScoreRequest>& requests, int k = 0) {
    const int d = weights_.config.d_model;
    const size_t T = 1 + weights_.config.head_specs.size();
    std::vector<Packed> ps;
    std::vector<Out> os;
    ps.reserve(requests.size());
    os.reserve(requests.size());
    std::vector<sr_request> reqs;
    std::vector<sr_result> res;
    for (const auto& r : requests) {
      ps.emplace_back(r, d);
      os.emplace_back(r.items.size(), T, k);
    }
    for (size_t i = 0; i < requests.size(); ++i) {
      reqs.push_back(ps[i].req);
      res.push_back(os[i].res);
    }
    check(sr_engine_score_batch(e_.get(), reqs.data(), static_cast<int32_t>(reqs.size()),
                                res.data()));
    std::vector<ScoreResult> out;
    for (size_t i = 0; i < requests.size(); ++i) {
      os[i].res = res[i];  // k_returned / flops written by the call
      out.push_back(os[i].result(requests[i], weights_.config));
    }
    return out;
  }

  // Mixed items from compact retrieval embeddings (north_star (d)):
  // set_projection(P [d_emb x n_soft*d_model], n_soft) once, then
  // score_embeddings(..., EmbForm::Project) builds n_soft soft rows per item on
  // the device; EmbForm::Pad is the service's one zero-padded row per item
  // (service.cpp:208-217). Item i's id is item_ids[i] (default: its index).
  enum class EmbForm { Pad = SR_EMB_PAD, Project = SR_EMB_PROJECT };
  // Workspace for passes of up to `rows` packed rows (sr_engine_reserve).
  void reserve(std::int64_t rows) { check(sr_engine_reserve(e_.get(), rows)); }
  void set_projection(const std::vector<float>& proj, int d_emb, int n_soft) {
    check(sr_engine_set_projection(e_.get(), proj.empty() ? nullptr : proj.data(), d_emb,
                                   n_soft));
  }
  ScoreResult score_embeddings(const std::string& request_id, const std::vector<int>& prefix,
                               const std::vector<float>& emb, int d_emb, EmbForm form, int k = 0,
                               const std::vector<std::int64_t>& item_ids = {}) {
    if (d_emb < 1 || emb.size() % static_cast<size_t>(d_emb) != 0)
      throw Error(ErrorCode::PayloadInvalid, "embeddings are not [n x d_emb]");
    const size_t n = emb.size() / static_cast<size_t>(d_emb);
    std::vector<std::int64_t> ids = item_ids;
    if (ids.empty())
      for (size_t i = 0; i < n; ++i) ids.push_back(static_cast<std::int64_t>(i));
    std::vector<int32_t> pre(prefix.begin(), prefix.end());
    const size_t T = 1 + weights_.config.head_specs.size();
    ScoreRequest shape;  // ids / order for the result
    shape.request_id = request_id;
    shape.mode = ScoreMode::Mixed;
    for (size_t i = 0; i < n; ++i) {
      ScoreItem it;
      it.id = std::to_string(ids[i]);
      shape.items.push_back(std::move(it));
    }
    Out o(n, T, k);
    check(sr_engine_score_emb(e_.get(), pre.data(), static_cast<int32_t>(pre.size()), emb.data(),
                              d_emb, static_cast<int32_t>(n), ids.data(),
                              static_cast<int32_t>(form), &o.res));
    return o.result(shape, weights_.config);
  }

  // The service's output side on the device (service.cpp:242-277): calibrated
  // relevance from a fitted isotonic head (calibration.cpp:65-88) and the
  // optional score blend (task -> weight, applied in task-name order like the
  // reference's std::map); the top-k then ranks by the final score, available
  // per item through final_scores(). An empty head and blend turn it off.
  struct CalibrationBlock {  // calibration.hpp:18-23
    double lo = 0, hi = 0, value = 0;
  };
  void set_postprocess(const std::vector<CalibrationBlock>& head,
                       const std::map<std::string, double>& blend = {}) {
    std::vector<double> lo, hi, val;
    for (const auto& b : head) {
      lo.push_back(b.lo);
      hi.push_back(b.hi);
      val.push_back(b.value);
    }
    std::vector<int32_t> task;
    std::vector<double> w;
    for (const auto& [name, weight] : blend) {  // std::map: task-name order
      int32_t t = -1;
      if (name == kRelevanceTask) t = 0;
      for (size_t h = 0; h < weights_.config.head_specs.size() && t < 0; ++h)
        if (weights_.config.head_specs[h].name == name) t = static_cast<int32_t>(h + 1);
      if (t < 0) throw Error(ErrorCode::Alignment, "blend references unknown task: " + name);
      task.push_back(t);
      w.push_back(weight);
    }
    check(sr_engine_set_postprocess(e_.get(), lo.empty() ? nullptr : lo.data(),
                                    hi.empty() ? nullptr : hi.data(),
                                    val.empty() ? nullptr : val.data(),
                                    static_cast<int32_t>(lo.size()),
                                    task.empty() ? nullptr : task.data(),
                                    w.empty() ? nullptr : w.data(),
                                    static_cast<int32_t>(task.size())));
  }
  // Final (calibrated / blended) scores of the last score call, item order.
  std::vector<double> final_scores(size_t n_items) {
    std::vector<double> out(n_items > 0 ? n_items : 1);
    int32_t got = 0;
    check(sr_engine_final_scores(e_.get(), out.data(), static_cast<int32_t>(out.size()), &got));
    out.resize(static_cast<size_t>(got));
    return out;
  }

  // This rank's shard (items with global ids) scored and merged across the
  // ranks of `comm`: every rank returns the global top-k; `items` holds this
  // shard's scores only.
  ScoreResult score_sharded(Comm& comm, const ScoreRequest& shard, int k) {
    Packed p(shard, weights_.config.d_model);
    if (!p.numeric_ids)
      throw Error(ErrorCode::SpecViolation, "sharded scoring needs integer (global) item ids");
    Out o(shard.items.size(), 1 + weights_.config.head_specs.size(), k);
    check(sr_engine_score_sharded(e_.get(), comm.handle(), &p.req, &o.res));
    ScoreResult r = o.result(shard, weights_.config, /*topk_from_items=*/false);
    for (int j = 0; j < o.res.k_returned; ++j)
      r.topk.push_back({std::to_string(o.tid[j]), o.tsc[j]});
    return r;
  }

  // handle_search's cache probe -> score misses -> put (service.cpp:160-234),
  // then the page ranking on the device. Item ids must be integers (the cache
  // keys' entity ids); *hits receives the number of cached items.
  ScoreResult score_cached(const ScoreRequest& request, ScoreCache& cache,
                           const std::string& searcher_id, std::uint64_t signature, int k = 0,
                           int* hits = nullptr) {
    Packed p(request, weights_.config.d_model);
    if (!p.numeric_ids)
      throw Error(ErrorCode::SpecViolation, "cached scoring needs integer item ids");
    Out o(request.items.size(), 1 + weights_.config.head_specs.size(), k);
    int32_t h = 0;
    check(sr_engine_score_cached(e_.get(), cache.handle(), searcher_id.c_str(), signature,
                                 weights_.version.c_str(), &p.req, &o.res, &h));
    if (hits) *hits = h;
    return o.result(request, weights_.config);
  }

 private:
  struct Packed {  // sr_request over the request's flattened arrays
    std::vector<int32_t> prefix, off{0}, toks;
    std::vector<float> rows;
    std::vector<int64_t> ids;
    bool numeric_ids = true;
    sr_request req{};
    Packed(const ScoreRequest& request, int d) : Packed(request, d, request.mode) {}
    Packed(const ScoreRequest& request, int d, ScoreMode mode) {
      const bool mixed = mode == ScoreMode::Mixed;
      prefix.assign(request.prefix_tokens.begin(), request.prefix_tokens.end());
      for (const auto& it : request.items) {
        if (mixed) {
          if (it.n_emb_tokens < 1 ||
              it.embedding.size() != static_cast<size_t>(it.n_emb_tokens) * d)
            throw Error(ErrorCode::PayloadInvalid, "item " + it.id +
                                                       " embedding payload is not [n x " +
                                                       std::to_string(d) + "]");
          rows.insert(rows.end(), it.embedding.begin(), it.embedding.end());
          off.push_back(off.back() + it.n_emb_tokens);
        } else {
          toks.insert(toks.end(), it.tokens.begin(), it.tokens.end());
          off.push_back(off.back() + static_cast<int32_t>(it.tokens.size()));
        }
        try {
          size_t pos = 0;
          ids.push_back(std::stoll(it.id, &pos));
          numeric_ids = numeric_ids && pos == it.id.size();
        } catch (...) {
          numeric_ids = false;
        }
      }
      req = sr_request{prefix.data(), static_cast<int32_t>(prefix.size()),
                       static_cast<int32_t>(request.items.size()), off.data(),
                       toks.empty() ? nullptr : toks.data(), rows.empty() ? nullptr : rows.data(),
                       numeric_ids ? ids.data() : nullptr, static_cast<int32_t>(mode)};
    }
  };
  struct Out {  // caller-side result buffers
    size_t T;
    std::vector<double> scores, tsc;
    std::vector<int64_t> tid;
    std::vector<int32_t> tix;
    sr_result res{};
    Out(size_t n, size_t tasks, int k)
        : T(tasks), scores(n * tasks), tsc(k > 0 ? k : 1), tid(k > 0 ? k : 1),
          tix(k > 0 ? k : 1) {
      res = sr_result{scores.data(), k, tid.data(), tsc.data(), tix.data(), {}, 0, 0};
    }
    ScoreResult result(const ScoreRequest& request, const ModelConfig& cfg,
                       bool topk_from_items = true) const {
      ScoreResult out;
      out.request_id = request.request_id;
      out.mode = request.mode;
      out.flops = {res.flops.attention_units, res.flops.linear_units, res.flops.t_q,
                   res.flops.t_i_mean, res.flops.n_items};
      out.kv_incremental_per_item = res.kv_incremental_per_item;
      for (size_t i = 0; i < request.items.size(); ++i) {
        ItemScores s{request.items[i].id, {}};
        s.tasks[kRelevanceTask] = scores[i * T];
        for (size_t h = 1; h < T; ++h) s.tasks[cfg.head_specs[h - 1].name] = scores[i * T + h];
        out.items.push_back(std::move(s));
      }
      if (topk_from_items)
        for (int j = 0; j < res.k_returned; ++j)
          out.topk.push_back({request.items[tix[j]].id, tsc[j]});
      return out;
    }
  };

  struct Del {
    void operator()(sr_engine* e) const { sr_engine_destroy(e); }
  };
  ModelWeights weights_;
  std::unique_ptr<sr_engine, Del> e_;
  friend class Scheduler;
};

// Latency-bounded dynamic batching in front of one engine (sr_sched_*,
// SURVEY §8(f) row 1): any thread submits whole requests and waits on its
// ticket; one native dispatcher packs queued requests into device passes
// (plan_batches' FIFO rule, engine.cpp:278-326, plus a latency budget) — the
// replacement for callers serialising on ScoringEngine's mutex
// (engine.cpp:389-392). Requests are copied at submit.
class Scheduler {
 public:
  struct Options {
    int max_queries = 8;                    // requests per device pass
    std::int64_t max_rows = std::int64_t(1) << 22;  // packed rows per pass
    double budget_ms = 0.0;                 // latency rule (0 = off)
    int max_wait_us = 0;                    // hold an unfilled pass this long
    int k = 10;                             // top-k per request
    std::int64_t sat_rows = 0;              // requests this large run alone (0 = off)
  };
  struct Stats {
    std::int64_t submitted = 0, completed = 0, failed = 0, batches = 0;
    double mean_batch = 0, p50_ms = 0, p99_ms = 0, max_ms = 0, mean_ms = 0;
  };

  Scheduler(ScoringEngine& engine, const Options& o) : engine_(engine), k_(o.k) {
    sr_sched_options so{o.max_queries, o.max_rows, o.budget_ms, o.max_wait_us, o.k, 0, o.sat_rows};
    sr_sched* s = nullptr;
    check(sr_sched_create(engine.e_.get(), &so, &s));
    s_.reset(s);
  }

  std::uint64_t submit(const ScoreRequest& request) {
    ScoringEngine::Packed p(request, engine_.weights_.config.d_model);
    std::uint64_t t = 0;
    check(sr_sched_submit(s_.get(), &p.req, &t));  // deep-copied by the dispatcher
    std::lock_guard<std::mutex> lock(mu_);
    pending_.emplace(t, request);
    return t;
  }

  // Blocks until the ticket's pass is done; rethrows the request's own error.
  ScoreResult wait(std::uint64_t ticket, double* latency_ms = nullptr) {
    ScoreRequest request;
    {
      std::lock_guard<std::mutex> lock(mu_);
      auto it = pending_.find(ticket);
      if (it == pending_.end()) throw Error(ErrorCode::StateInvalid, "unknown ticket");
      request = std::move(it->second);
      pending_.erase(it);
    }
    ScoringEngine::Out o(request.items.size(), 1 + engine_.weights_.config.head_specs.size(), k_);
    double lat = 0;
    int32_t nq = 0;
    check(sr_sched_wait(s_.get(), ticket, &o.res, &lat, &nq));
    if (latency_ms) *latency_ms = lat;
    return o.result(request, engine_.weights_.config);
  }

  Stats stats(bool reset = false) {
    sr_sched_stats st{};
    check(sr_sched_get_stats(s_.get(), reset ? 1 : 0, &st));
    return {st.submitted, st.completed, st.failed, st.batches, st.mean_batch,
            st.p50_ms, st.p99_ms, st.max_ms, st.mean_ms};
  }

 private:
  struct Del {
    void operator()(sr_sched* s) const { sr_sched_destroy(s); }
  };
  ScoringEngine& engine_;
  int k_;
  std::mutex mu_;
  std::map<std::uint64_t, ScoreRequest> pending_;
  std::unique_ptr<sr_sched, Del> s_;  // destroyed first: joins the dispatcher
};

inline ScoreResult score_by_mode(ScoringEngine& engine, const ScoreRequest& request) {
  return engine.score(request);  // engine.cpp:379-387
}

// ------------------------------------------- reference free functions
// engine.hpp:77-89 take the weights, not an engine. Each ModelWeights handle
// gets one process-wide ScoringEngine on the default device (created on first
// use, kept for the handle's lifetime in this process), so callers such as
// semrank_main.cpp:293/376/657 and acceptance_main.cpp:90-174 relink
// unchanged. ScoringEngine serialises calls on it (engine.cpp:389-392).
namespace detail {
inline int& default_device() {
  static int d = 0;
  return d;
}
inline ScoringEngine& engine_for(const ModelWeights& w) {
  static std::mutex mu;
  static std::map<const sr_weights*, std::unique_ptr<ScoringEngine>> engines;
  std::lock_guard<std::mutex> lock(mu);
  auto& e = engines[w.handle()];
  if (!e) e = std::make_unique<ScoringEngine>(w, default_device());
  return *e;
}
}  // namespace detail

// Device used by the weights-level functions below (default 0).
inline void set_default_device(int device) { detail::default_device() = device; }

inline ScoreResult score_naive(const ModelWeights& w, const ScoreRequest& r) {
  return detail::engine_for(w).score_as(r, ScoreMode::Naive);
}
inline ScoreResult score_ibpc(const ModelWeights& w, const ScoreRequest& r) {
  return detail::engine_for(w).score_as(r, ScoreMode::Ibpc);
}
// One pass: the whole packed sequence must fit max_seq (engine.cpp:189-200);
// when it fits, the chunked accounting below is the single-pass one.
inline ScoreResult score_multi_item(const ModelWeights& w, const ScoreRequest& r) {
  long total = static_cast<long>(r.prefix_tokens.size());
  for (const auto& it : r.items) total += static_cast<long>(it.tokens.size());
  if (total > w.config.max_seq)
    throw Error(ErrorCode::LengthOverflow,
                "multi-item sequence of " + std::to_string(total) + " exceeds max_seq " +
                    std::to_string(w.config.max_seq) + "; split the request into smaller batches");
  return detail::engine_for(w).score_as(r, ScoreMode::MultiItem);
}
// No prefix re-payment on the device (the packed pass has no max_seq chunk
// limit); FlopReport still reports the reference's chunked accounting.
inline ScoreResult score_multi_item_chunked(const ModelWeights& w, const ScoreRequest& r) {
  return detail::engine_for(w).score_as(r, ScoreMode::MultiItem);
}
inline ScoreResult score_mixed(const ModelWeights& w, const ScoreRequest& r) {
  return detail::engine_for(w).score_as(r, ScoreMode::Mixed);
}
inline ScoreResult score_by_mode(const ModelWeights& w, const ScoreRequest& r) {
  return detail::engine_for(w).score(r);  // engine.cpp:379-387
}

// ------------------------------------------------ prompt + /score body
struct PromptParts {  // prompt.hpp:17-20
  std::vector<int> prefix_tokens;
  std::vector<int> item_tokens;
};
inline constexpr const char* kPromptSuffix = "\nRelevant (Yes/No): ";  // prompt.hpp:23

inline PromptParts build_prompt(const std::string& system, const std::string& query_context,
                                const std::string& document, int max_seq = 4096) {
  int32_t np = 0, ni = 0;
  check(sr_build_prompt(system.data(), static_cast<int64_t>(system.size()), query_context.data(),
                        static_cast<int64_t>(query_context.size()), document.data(),
                        static_cast<int64_t>(document.size()), max_seq, nullptr, 0, &np, nullptr,
                        0, &ni));
  std::vector<int32_t> p(static_cast<size_t>(np)), it(static_cast<size_t>(ni));
  check(sr_build_prompt(system.data(), static_cast<int64_t>(system.size()), query_context.data(),
                        static_cast<int64_t>(query_context.size()), document.data(),
                        static_cast<int64_t>(document.size()), max_seq, p.data(), np, &np,
                        it.data(), ni, &ni));
  return {std::vector<int>(p.begin(), p.end()), std::vector<int>(it.begin(), it.end())};
}

// service.cpp:380-391, byte-identical to the reference's nlohmann dump().
inline std::string score_result_to_json(const ScoreResult& result) {
  std::vector<const char*> ids, names;
  std::vector<double> scores;
  if (!result.items.empty())
    for (const auto& [name, v] : result.items[0].tasks) names.push_back(name.c_str());
  for (const auto& it : result.items) {
    ids.push_back(it.item_id.c_str());
    for (const char* n : names) scores.push_back(it.tasks.at(n));
  }
  const sr_flop_report fl{result.flops.attention_units, result.flops.linear_units,
                          result.flops.t_q, result.flops.t_i_mean, result.flops.n_items};
  int64_t len = 0;
  const auto n_items = static_cast<int32_t>(ids.size());
  const auto n_tasks = static_cast<int32_t>(names.size());
  check(sr_score_result_to_json(result.request_id.c_str(), n_items, ids.data(), n_tasks,
                                names.data(), scores.data(), &fl, nullptr, 0, &len));
  std::string out(static_cast<size_t>(len), '\0');
  check(sr_score_result_to_json(result.request_id.c_str(), n_items, ids.data(), n_tasks,
                                names.data(), scores.data(), &fl, out.data(), len, &len));
  return out;
}

}  // namespace semrank
