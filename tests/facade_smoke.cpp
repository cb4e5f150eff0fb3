// Compiles a reference-style caller against the C++ facade
// (include/semrank_b200.hpp) and exercises the host-side API. Built and run by
// tests/test_facade.py; with a GPU present it also scores one request.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "semrank_b200.hpp"

int main(int argc, char** argv) {
  using namespace semrank;
  const auto cfg = ModelConfig::default_toy();
  cfg.validate();
  const auto f = flops(ScoreMode::Ibpc, 500, 50, 100);  // engine.cpp:30-47
  if (f.attention_units != 5500000.0) return 2;
  auto w = init_model(cfg, 1);
  if (w.version != "toy-0000000000000001") return 3;
  try {
    ModelConfig bad = cfg;
    bad.d_model = 65;
    bad.validate();
    return 4;
  } catch (const Error& e) {
    if (e.code() != ErrorCode::SpecViolation) return 5;
  }
  // mid-tier cache (test_midtier.cpp:18-56; signature from tests/golden/score_cache.json)
  const auto canon = canonical_query("Senior  ML Engineer ", {{"region", {"na", "emea"}}});
  if (canon != "senior ml engineer|region=emea,na") return 7;
  if (fnv1a64(canon) != 9702648040046958735ull) return 8;
  {
    ScoreCache cache(2, {"relevance"});
    const CacheKey ka{"s", 1, 1, "v"}, kb{"s", 1, 2, "v"}, kc{"s", 1, 3, "v"};
    if (cache.get(ka)) return 9;
    cache.put(ka, {{"relevance", 0.9}});
    if (!cache.get(ka) || cache.get(ka)->at("relevance") != 0.9) return 10;
    cache.put(kb, {{"relevance", 0.5}});
    cache.put(kc, {{"relevance", 0.1}});
    if (cache.size() != 2 || cache.get(ka) || !cache.get(kb) || !cache.get(kc)) return 11;
    try {
      cache.put(kb, {{"relevance", 0.6}});
      return 12;
    } catch (const Error& e) {
      if (e.code() != ErrorCode::Consistency) return 13;
    }
  }
  if (argc > 1 && std::string(argv[1]) == "gpu") {
    ScoringEngine engine(w, 0);
    engine.reserve(4096);  // the serving warm-up order: workspace first
    ScoreRequest req;
    req.request_id = "facade";
    req.mode = ScoreMode::MultiItem;
    for (int i = 0; i < 20; ++i) req.prefix_tokens.push_back(i);
    for (int j = 0; j < 4; ++j) {
      ScoreItem it;
      it.id = std::to_string(100 + j);
      for (int t = 0; t < 5 + j; ++t) it.tokens.push_back(40 + t * j);
      req.items.push_back(it);
    }
    const auto r = engine.score(req, 2);
    if (r.items.size() != 4 || r.topk.size() != 2) return 6;
    ScoreCache cache(16);
    const auto sig = fnv1a64(canonical_query("nurse", {}));
    int hits = -1;
    const auto c1 = engine.score_cached(req, cache, "s", sig, 2, &hits);
    if (hits != 0 || cache.size() != 4) return 14;
    const auto c2 = engine.score_cached(req, cache, "s", sig, 2, &hits);
    if (hits != 4) return 15;
    for (int i = 0; i < 4; ++i)
      if (c1.items[i].tasks != r.items[i].tasks || c2.items[i].tasks != r.items[i].tasks) return 16;
    if (c2.topk != r.topk) return 17;
    {
      // batched pass: each request's scores within the bf16 tolerance of its own pass
      ScoreRequest req2 = req;
      req2.request_id = "facade2";
      req2.items.pop_back();
      const auto both = engine.score_batch({req, req2}, 2);
      if (both.size() != 2 || both[0].items.size() != 4 || both[1].items.size() != 3) return 21;
      for (int i = 0; i < 3; ++i)
        if (std::abs(both[1].items[i].tasks.at(kRelevanceTask) -
                     r.items[i].tasks.at(kRelevanceTask)) > 6e-3)
          return 22;
      // compact embeddings: service zero-pad form and a device projection
      const int d_emb = 16, n_soft = 2, d = cfg.d_model;
      std::vector<float> emb(3 * d_emb);
      for (size_t i = 0; i < emb.size(); ++i) emb[i] = 0.01f * static_cast<float>(i % 7);
      const auto pad = engine.score_embeddings("pad", req.prefix_tokens, emb, d_emb,
                                               ScoringEngine::EmbForm::Pad, 2, {7, 8, 9});
      if (pad.items.size() != 3 || pad.items[0].item_id != "7" || pad.topk.size() != 2) return 23;
      std::vector<float> proj(static_cast<size_t>(d_emb) * n_soft * d, 0.001f);
      engine.set_projection(proj, d_emb, n_soft);
      const auto pr = engine.score_embeddings("proj", req.prefix_tokens, emb, d_emb,
                                              ScoringEngine::EmbForm::Project, 2);
      if (pr.items.size() != 3 || pr.kv_incremental_per_item != n_soft) return 24;
    }
    {
      // service post-processing: a two-block isotonic head and a blend
      engine.set_postprocess({{0.0, 0.5, 0.2}, {0.5, 1.0, 0.9}},
                             {{"relevance", 1.0}, {"click", 0.5}});
      const auto pp = engine.score(req, 2);
      const auto fin = engine.final_scores(req.items.size());
      if (fin.size() != 4 || pp.topk.size() != 2) return 25;
      for (int i = 0; i < 4; ++i) {
        const double rel = pp.items[i].tasks.at(kRelevanceTask);
        const double cal = rel <= 0.5 ? 0.2 : 0.9;  // calibration.cpp:69-85
        if (std::abs(fin[i] - (cal + 0.5 * pp.items[i].tasks.at("click"))) > 1e-9) return 26;
      }
      try {
        engine.set_postprocess({}, {{"relevance", 1.0}});  // blend without a fitted head
        return 27;
      } catch (const Error& e) {
        if (e.code() != ErrorCode::StateInvalid) return 28;
      }
      engine.set_postprocess({});
    }
    {
      // candidate sharding through NCCL at one rank: the merged top-k is the
      // single-GPU top-k (global ids = the items' numeric ids)
      Comm comm(1, 0, Comm::unique_id(), 0);
      const auto sh = engine.score_sharded(comm, req, 2);
      if (sh.topk != r.topk) return 29;
    }
    {
      // retrieval top-K: 50 docs, d_emb 4, one feature; ties by doc id
      std::vector<float> embv, feat;
      std::vector<std::int64_t> ids;
      for (int i = 0; i < 50; ++i) {
        for (int j = 0; j < 4; ++j) embv.push_back(1.0f + 0.01f * static_cast<float>((i * 7 + j) % 11));
        feat.push_back(static_cast<float>(i % 5));
        ids.push_back(1000 - i);
      }
      Corpus corpus(embv, feat, ids, 4, 1, 0);
      const auto top = corpus.topk({1.f, 1.f, 1.f, 1.f}, 1.0, {0.1}, 5);
      if (top.size() != 5) return 30;
      for (size_t i = 1; i < top.size(); ++i)
        if (top[i - 1].score < top[i].score ||
            (top[i - 1].score == top[i].score && top[i - 1].doc_id > top[i].doc_id))
          return 31;
    }
    {
      // the serving scheduler: concurrent-style submit / wait, each result
      // identical to scoring the request alone (one request per pass here)
      Scheduler::Options so;
      so.max_queries = 4;
      so.k = 2;
      Scheduler sched(engine, so);
      std::vector<std::uint64_t> tickets;
      for (int q = 0; q < 3; ++q) tickets.push_back(sched.submit(req));
      for (auto t : tickets) {
        double lat = -1;
        const auto s = sched.wait(t, &lat);
        if (s.items.size() != 4 || s.topk != r.topk || lat < 0) return 18;
        for (int i = 0; i < 4; ++i)
          if (std::abs(s.items[i].tasks.at(kRelevanceTask) - r.items[i].tasks.at(kRelevanceTask)) >
              6e-3)
            return 19;
      }
      if (sched.stats().completed != 3) return 20;
    }
    std::printf("relevance[0]=%.6f top=%s\n", r.items[0].tasks.at(kRelevanceTask),
                r.topk[0].first.c_str());
  }
  std::printf("facade ok\n");
  return 0;
}
