// Compiles a reference-style caller against the C++ facade
// (include/semrank_b200.hpp) and exercises the host-side API. Built and run by
// tests/test_facade.py; with a GPU present it also scores one request.
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
  if (argc > 1 && std::string(argv[1]) == "gpu") {
    ScoringEngine engine(w, 0);
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
    std::printf("relevance[0]=%.6f top=%s\n", r.items[0].tasks.at(kRelevanceTask),
                r.topk[0].first.c_str());
  }
  std::printf("facade ok\n");
  return 0;
}
