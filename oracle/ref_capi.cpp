// ref_capi.cpp — C harness around the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY (see oracle/semrank_oracle.c header). Built by
// oracle/Makefile together with /root/reference/proj/src/{model,kernels,
// engine,tokenizer,error,weights_io,prompt}.cpp compiled in place into
// oracle/_ref/libsemrank_ref.so. Used to (a) generate the golden vectors in
// tests/golden/, (b) pin the C restatement, (c) time the reference CPU path
// for bench.py's cpu_baseline / --impl reference arm. Nothing here is
// shipped or called by the product.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "semrank/engine.hpp"
#include "semrank/error.hpp"
#include "semrank/kernels.hpp"
#include "semrank/model.hpp"
#include "semrank/calibration.hpp"
#include "semrank/base64.hpp"
#include "semrank/retrieval.hpp"
#include "semrank/midtier.hpp"
#include "semrank/rng.hpp"
#include "semrank/weights_io.hpp"
#include "semrank/prompt.hpp"

#include <json.hpp>  // the nlohmann/json the reference serialises with (service.cpp:11)

using namespace semrank;

namespace {
thread_local std::string g_err;
std::mutex g_mu;
std::map<std::string, std::shared_ptr<ModelWeights>> g_weights;

std::shared_ptr<ModelWeights> weights_for(const char* path) {
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_weights.find(path);
  if (it != g_weights.end()) return it->second;
  auto w = std::make_shared<ModelWeights>(load_weights(path));
  g_weights[path] = w;
  return w;
}

ModelConfig make_config(const int32_t* dims, int32_t n_heads_task, const char* const* names,
                        const int32_t* arity) {
  ModelConfig c;
  c.n_layers = dims[0];
  c.d_model = dims[1];
  c.n_heads = dims[2];
  c.d_ff = dims[3];
  c.vocab_size = dims[4];
  c.max_seq = dims[5];
  c.yes_token_id = dims[6];
  c.no_token_id = dims[7];
  for (int i = 0; i < n_heads_task; ++i) c.head_specs.push_back({names[i], arity[i]});
  return c;
}

template <typename F>
int run(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_parallel(int parallel) {
  kernels::set_default_exec(parallel ? kernels::Exec::Parallel : kernels::Exec::Serial);
}

void ref_forget_weights() {
  std::lock_guard<std::mutex> lock(g_mu);
  g_weights.clear();
}

// dims = {n_layers, d_model, n_heads, d_ff, vocab_size, max_seq, yes, no}
int ref_init_save(const int32_t* dims, int32_t n_heads_task, const char* const* names,
                  const int32_t* arity, uint64_t seed, const char* path) {
  return run([&] {
    const auto w = init_model(make_config(dims, n_heads_task, names, arity), seed);
    save_weights(w, path);
  });
}

// Fan-in scaled variant, built with the reference's own Rng and
// container: same substream ("init"), same draw order as init_model
// (model.cpp:94-134), only the per-tensor std differs.
int ref_init_fanin_save(const int32_t* dims, int32_t n_heads_task, const char* const* names,
                        const int32_t* arity, uint64_t seed, const char* path) {
  return run([&] {
    const ModelConfig cfg = make_config(dims, n_heads_task, names, arity);
    cfg.validate();
    Rng rng = Rng::substream(seed, "init");
    ModelWeights w;
    w.config = cfg;
    char buf[40];
    std::snprintf(buf, sizeof(buf), "fanin-%016llx", static_cast<unsigned long long>(seed));
    w.version = buf;
    auto fill = [&](std::vector<float>& t, size_t n, double sd) {
      t.resize(n);
      for (auto& v : t) v = static_cast<float>(std::clamp(rng.normal(0.0, sd), -1.0, 1.0));
    };
    const size_t d = cfg.d_model, F = cfg.d_ff;
    const double e = static_cast<double>(0.08f);
    const double resid = std::sqrt(2.0 * cfg.n_layers);
    const double sd = 1.0 / std::sqrt(static_cast<double>(d));
    fill(w.tok_emb, static_cast<size_t>(cfg.vocab_size) * d, e);
    fill(w.pos_emb, static_cast<size_t>(cfg.max_seq) * d, e);
    w.layers.resize(cfg.n_layers);
    for (auto& l : w.layers) {
      fill(l.wq, d * d, sd);
      fill(l.wk, d * d, sd);
      fill(l.wv, d * d, sd);
      fill(l.wo, d * d, sd / resid);
      l.ln1_gain.assign(d, 1.0f);
      l.ln2_gain.assign(d, 1.0f);
      fill(l.w_mlp_in, d * F, sd);
      fill(l.w_mlp_out, F * d, 1.0 / std::sqrt(static_cast<double>(F)) / resid);
    }
    w.ln_f_gain.assign(d, 1.0f);
    fill(w.w_vocab, d * static_cast<size_t>(cfg.vocab_size), sd);
    for (const auto& s : cfg.head_specs) {
      TaskHead h;
      h.name = s.name;
      h.arity = s.arity;
      fill(h.w, d * static_cast<size_t>(s.arity), sd);
      h.b.assign(s.arity, 0.0f);
      w.heads.push_back(std::move(h));
    }
    save_weights(w, path);
  });
}

// score_by_mode (engine.cpp:379-387) on a flattened request.
// scores_out: [n_items x (1 + n_heads)] = relevance, then heads in config order.
// flops_out: 5 doubles (FlopReport); kv_out: kv_incremental_per_item.
int ref_score(const char* weights_path, int32_t mode, const int32_t* prefix, int32_t t_q,
              const int32_t* offsets, const int32_t* tokens, const float* rows, int32_t n_items,
              double* scores_out, double* flops_out, double* kv_out) {
  return run([&] {
    const auto w = weights_for(weights_path);
    const int d = w->config.d_model;
    ScoreRequest req;
    req.request_id = "ref";
    req.prefix_tokens.assign(prefix, prefix + t_q);
    req.mode = static_cast<ScoreMode>(mode);
    for (int i = 0; i < n_items; ++i) {
      ScoreItem it;
      it.id = std::to_string(i);
      if (req.mode == ScoreMode::Mixed) {
        it.n_emb_tokens = offsets[i + 1] - offsets[i];
        it.embedding.assign(rows + static_cast<size_t>(offsets[i]) * d,
                            rows + static_cast<size_t>(offsets[i + 1]) * d);
      } else {
        it.tokens.assign(tokens + offsets[i], tokens + offsets[i + 1]);
      }
      req.items.push_back(std::move(it));
    }
    const ScoreResult r = score_by_mode(*w, req);
    const int T = 1 + static_cast<int>(w->config.head_specs.size());
    for (int i = 0; i < n_items; ++i) {
      const auto& tasks = r.items[i].tasks;
      scores_out[static_cast<size_t>(i) * T] = tasks.at(kRelevanceTask);
      for (size_t h = 0; h < w->config.head_specs.size(); ++h)
        scores_out[static_cast<size_t>(i) * T + 1 + h] = tasks.at(w->config.head_specs[h].name);
    }
    if (flops_out) {
      flops_out[0] = r.flops.attention_units;
      flops_out[1] = r.flops.linear_units;
      flops_out[2] = r.flops.t_q;
      flops_out[3] = r.flops.t_i_mean;
      flops_out[4] = r.flops.n_items;
    }
    if (kv_out) *kv_out = r.kv_incremental_per_item;
  });
}

// prefill (model.cpp:251-273) from an empty cache; out_rows [n x d].
int ref_prefill(const char* weights_path, const int32_t* tokens, int32_t n, float* out_rows) {
  return run([&] {
    const auto w = weights_for(weights_path);
    KVCache cache = KVCache::empty(w->config);
    std::vector<int> t(tokens, tokens + n);
    const auto h = prefill(*w, t, cache);
    std::memcpy(out_rows, h.data(), h.size() * sizeof(float));
  });
}

// kernels::attention_serial (kernels.cpp:175-192); spans3 = {prefix_end, span_start, pos}.
void ref_attention(const float* q, const float* k, const float* v, float* out, int32_t n_new,
                   int32_t n_heads, int32_t head_dim, const int32_t* spans3) {
  std::vector<kernels::MaskSpan> spans(n_new);
  for (int i = 0; i < n_new; ++i) spans[i] = {spans3[3 * i], spans3[3 * i + 1], spans3[3 * i + 2]};
  kernels::attention_serial(q, k, v, out, n_new, n_heads, head_dim, spans.data());
}

int ref_flops(int32_t mode, int64_t t_q, int64_t t_i, int64_t n, double* out5) {
  return run([&] {
    const auto r = flops(static_cast<ScoreMode>(mode), t_q, t_i, n);
    out5[0] = r.attention_units;
    out5[1] = r.linear_units;
    out5[2] = r.t_q;
    out5[3] = r.t_i_mean;
    out5[4] = r.n_items;
  });
}

// plan_batches (engine.cpp:278-326) -> (batch, request, begin, end) quadruples.
int ref_plan_batches(int32_t n_req, const int32_t* prefix_len, const int32_t* req_item_off,
                     const int32_t* item_len, int64_t budget, int32_t* out, int32_t cap,
                     int32_t* n_out, int64_t* tokens_out) {
  return run([&] {
    std::vector<ScoreRequest> reqs(n_req);
    for (int r = 0; r < n_req; ++r) {
      reqs[r].prefix_tokens.assign(prefix_len[r], 1);
      for (int i = req_item_off[r]; i < req_item_off[r + 1]; ++i) {
        ScoreItem it;
        it.tokens.assign(item_len[i], 2);
        reqs[r].items.push_back(it);
      }
    }
    const auto plan = plan_batches(reqs, budget);
    int n = 0;
    for (size_t b = 0; b < plan.size(); ++b) {
      tokens_out[b] = plan[b].token_count;
      for (const auto& e : plan[b].entries) {
        if (n < cap) {
          out[4 * n] = static_cast<int32_t>(b);
          out[4 * n + 1] = static_cast<int32_t>(e.request_index);
          out[4 * n + 2] = static_cast<int32_t>(e.item_begin);
          out[4 * n + 3] = static_cast<int32_t>(e.item_end);
        }
        ++n;
      }
    }
    *n_out = n;
  });
}

// Rng(seed).uniform_int stream (rng.hpp:44-47), for seeded test requests.
void ref_uniform_ints(uint64_t seed, int64_t lo, int64_t hi, int32_t n, int64_t* out) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.uniform_int(lo, hi);
}

// exhaustive_topk (retrieval.cpp:134-173) on a columnar corpus. Each doc gets
// attribute "color" = kColors[color[i]]; allowed >= 0 colors form the query's
// filter (QuerySpec.filters["color"]), n_allowed < 0 means no filter, so the
// reference's own filter_candidates runs. Results: min(k, #candidates).
int ref_exhaustive_topk(const float* emb, const float* feat, const int64_t* ids,
                        const int32_t* color, int64_t n, int32_t d, int32_t f,
                        const float* query, int32_t d_query, double w0, const double* w,
                        int32_t n_w, const int32_t* allowed, int32_t n_allowed, int32_t k,
                        int64_t* ids_out, double* scores_out, int32_t* n_out, double* secs_out) {
  static const char* kColors[] = {"red", "blue", "green", "black", "white", "grey", "pink",
                                  "teal"};
  return run([&] {
    Corpus corpus;
    for (int j = 0; j < f; ++j) corpus.feature_names.push_back("f" + std::to_string(j));
    corpus.docs.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
      DocumentRecord& doc = corpus.docs[static_cast<size_t>(i)];
      doc.doc_id = ids[i];
      if (color != nullptr) doc.attributes["color"] = kColors[color[i] & 7];
      doc.embedding.assign(emb + i * d, emb + (i + 1) * d);
      doc.features.assign(feat + i * f, feat + (i + 1) * f);
    }
    QuerySpec q;
    q.embedding.assign(query, query + d_query);
    q.k = k;
    if (n_allowed >= 0) {
      auto& v = q.filters["color"];
      for (int j = 0; j < n_allowed; ++j) v.push_back(kColors[allowed[j] & 7]);
    }
    RARWeights rw;
    rw.w0 = w0;
    rw.w.assign(w, w + n_w);
    const auto t0 = std::chrono::steady_clock::now();
    const auto top = exhaustive_topk(corpus, q, rw, kernels::default_exec());
    if (secs_out)
      *secs_out = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (size_t j = 0; j < top.size(); ++j) {
      ids_out[j] = top[j].doc_id;
      scores_out[j] = top[j].score;
    }
    *n_out = static_cast<int32_t>(top.size());
  });
}

// fit_isotonic (calibration.cpp:13-63) on (raw, outcome) pairs, then
// calibrate (:65-88) of raws[]; blocks written to lo/hi/val (cap entries).
int ref_fit_calibrate(const double* raw, const int32_t* outcome, int32_t n, const double* raws,
                      int32_t n_raws, double* lo, double* hi, double* val, int32_t cap,
                      int32_t* n_blocks, double* out) {
  return run([&] {
    std::vector<CalibrationPair> pairs(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) pairs[i] = {raw[i], outcome[i]};
    const auto head = fit_isotonic(pairs);
    *n_blocks = static_cast<int32_t>(head.blocks.size());
    for (size_t b = 0; b < head.blocks.size() && static_cast<int32_t>(b) < cap; ++b) {
      lo[b] = head.blocks[b].lo;
      hi[b] = head.blocks[b].hi;
      val[b] = head.blocks[b].value;
    }
    for (int i = 0; i < n_raws; ++i) out[i] = calibrate(head, raws[i]);
  });
}

// decode_f32_base64 (base64.cpp:97-108); returns the reference's status
// (1 + ErrorCode) and message via ref_last_error on malformed payloads.
int ref_decode_f32_base64(const char* text, int64_t len, float* out, int64_t cap, int64_t* n_out) {
  return run([&] {
    const auto v = decode_f32_base64(std::string(text, static_cast<size_t>(len)));
    for (size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = v[i];
    *n_out = static_cast<int64_t>(v.size());
  });
}

// canonical_query (midtier.cpp:14-44) with filters given as (attr, value)
// pairs grouped into the reference's map<string, vector<string>>.
int ref_canonical_query(const char* text, int32_t n, const char* const* attrs,
                        const char* const* values, char* out, int64_t cap, int64_t* len,
                        uint64_t* fnv) {
  return run([&] {
    std::map<std::string, std::vector<std::string>> filters;
    for (int32_t i = 0; i < n; ++i) filters[attrs[i]].push_back(values[i]);
    const auto c = canonical_query(text, filters);
    std::memcpy(out, c.data(), std::min<size_t>(c.size(), static_cast<size_t>(cap)));
    *len = static_cast<int64_t>(c.size());
    *fnv = fnv1a64(c);
  });
}

// A scripted ScoreCache trace (midtier.cpp:64-100): op[i] 0 = get, 1 = put
// of {"relevance": value[i]} under key (searcher[i], sig[i], entity[i],
// version[i]). out_hit[i] = hit (get) / status (put, 1 + ErrorCode or 0),
// out_val[i] = the value a hit returned, out_size[i] = size() after the op.
int ref_cache_trace(int64_t capacity, int32_t n_ops, const int32_t* op,
                    const char* const* searcher, const uint64_t* sig, const int64_t* entity,
                    const char* const* version, const double* value, int32_t* out_hit,
                    double* out_val, int64_t* out_size) {
  return run([&] {
    ScoreCache cache(static_cast<std::size_t>(capacity));
    for (int32_t i = 0; i < n_ops; ++i) {
      const CacheKey key{searcher[i], sig[i], entity[i], version[i]};
      out_val[i] = 0.0;
      if (op[i] == 0) {
        const auto got = cache.get(key);
        out_hit[i] = got.has_value() ? 1 : 0;
        if (got) out_val[i] = got->at("relevance");
      } else {
        out_hit[i] = run([&] { cache.put(key, TaskScoreMap{{"relevance", value[i]}}); });
      }
      out_size[i] = static_cast<int64_t>(cache.size());
    }
  });
}

// build_prompt (prompt.cpp:14-38), the reference itself. Lengths written to
// n_out[0..1]; tokens up to cap each.
int ref_build_prompt(const char* system, const char* query, const char* document, int32_t max_seq,
                     int32_t* prefix_out, int32_t* item_out, int32_t cap, int32_t* n_out) {
  return run([&] {
    const auto parts = build_prompt(system, query, document, max_seq);
    n_out[0] = static_cast<int32_t>(parts.prefix_tokens.size());
    n_out[1] = static_cast<int32_t>(parts.item_tokens.size());
    for (int32_t i = 0; i < std::min<int32_t>(cap, n_out[0]); ++i) prefix_out[i] = parts.prefix_tokens[i];
    for (int32_t i = 0; i < std::min<int32_t>(cap, n_out[1]); ++i) item_out[i] = parts.item_tokens[i];
  });
}

// score_result_to_json lives in service.cpp, which cannot be built here
// (cpp-httplib is not vendored). Its body (service.cpp:380-391) is three
// nlohmann::json statements; they are restated here verbatim in structure
// over the same json library so the golden bytes come from the reference's
// serialiser. Result fields as a flattened ScoreResult.
int ref_score_result_json(const char* request_id, int32_t n_items, const char* const* ids,
                          int32_t n_tasks, const char* const* task_names, const double* scores,
                          double attention, double linear, char* out, int64_t cap, int64_t* len) {
  return run([&] {
    using json = nlohmann::json;
    json arr = json::array();
    for (int32_t i = 0; i < n_items; ++i) {
      std::map<std::string, double> tasks;
      for (int32_t t = 0; t < n_tasks; ++t) tasks[task_names[t]] = scores[i * n_tasks + t];
      arr.push_back({{"id", std::string(ids[i])}, {"tasks", tasks}});
    }
    const json j = {{"request_id", std::string(request_id)},
                    {"scores", arr},
                    {"flops", {{"attention", attention}, {"linear", linear}}}};
    const std::string s = j.dump();
    *len = static_cast<int64_t>(s.size());
    std::memcpy(out, s.data(), std::min<size_t>(static_cast<size_t>(cap), s.size()));
  });
}

}  // extern "C"
