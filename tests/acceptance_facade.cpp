// Acceptance criteria 1 and 4 of the reference (acceptance_main.cpp:90-104,
// 146-174) written exactly as the reference writes them — weights-level
// score_naive / score_ibpc / score_multi_item_chunked / score_mixed /
// score_by_mode and weights.tok_emb — but compiled against the C++ facade
// (include/semrank_b200.hpp) and linked with libsemrank_b200.so, so every
// call runs on the device. Plus the reference's text path around the scorer:
// build_prompt items (prompt.cpp:14-38) scored and rendered with
// score_result_to_json (service.cpp:380-391). Built and run by
// tests/test_facade.py (GPU).
#include <cmath>
#include <cstdio>
#include <string>

#include "semrank_b200.hpp"

using namespace semrank;

namespace {
// semrank::Rng (rng.hpp:33-47): splitmix64, uniform_int = lo + next % span.
struct Rng {
  std::uint64_t s;
  explicit Rng(std::uint64_t seed) : s(seed) {}
  std::uint64_t next() {
    s += 0x9E3779B97F4A7C15ull;
    std::uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  long uniform_int(long lo, long hi) {
    return lo + static_cast<long>(next() % static_cast<std::uint64_t>(hi - lo + 1));
  }
};

ScoreRequest seeded_request(Rng& rng, int t_q, int t_i, int n_items) {  // acceptance_main.cpp:62-76
  ScoreRequest req;
  for (int i = 0; i < t_q; ++i) req.prefix_tokens.push_back(static_cast<int>(rng.uniform_int(0, 255)));
  for (int i = 0; i < n_items; ++i) {
    ScoreItem item;
    item.id = std::to_string(i);
    for (int j = 0; j < t_i; ++j) item.tokens.push_back(static_cast<int>(rng.uniform_int(0, 255)));
    req.items.push_back(std::move(item));
  }
  return req;
}

double max_dev(const ScoreResult& a, const ScoreResult& b) {
  double dev = 0;
  for (std::size_t i = 0; i < a.items.size(); ++i)
    for (const auto& [task, p] : a.items[i].tasks)
      dev = std::max(dev, std::fabs(p - b.items[i].tasks.at(task)));
  return dev;
}

int fails = 0;
void criterion(int id, const char* what, bool ok, const std::string& detail) {
  std::printf("criterion %d %s: %s (%s)\n", id, ok ? "PASS" : "FAIL", what, detail.c_str());
  if (!ok) ++fails;
}
}  // namespace

int main() {
  const auto weights = init_model(ModelConfig::default_toy(), 2026);  // acceptance_main.cpp seed

  {  // criterion 1: mode equivalence on 20 seeded requests (1e-5)
    Rng rng(101);
    double dev_ibpc = 0, dev_multi = 0;
    for (int r = 0; r < 20; ++r) {
      const auto req = seeded_request(rng, 50, 150, 50);
      const auto naive = score_naive(weights, req);
      dev_ibpc = std::max(dev_ibpc, max_dev(naive, score_ibpc(weights, req)));
      dev_multi = std::max(dev_multi, max_dev(naive, score_multi_item_chunked(weights, req)));
    }
    char buf[160];
    std::snprintf(buf, sizeof(buf), "max |ibpc-naive| = %.2e, max |multi-naive| = %.2e, tol 1e-5",
                  dev_ibpc, dev_multi);
    criterion(1, "mode equivalence on 20 seeded requests", dev_ibpc <= 1e-5 && dev_multi <= 1e-5,
              buf);
  }
  {  // criterion 4: mixed-input equivalence and 1-token KV growth
    Rng rng(104);
    auto req = seeded_request(rng, 40, 12, 10);
    ScoreRequest mixed = req;
    mixed.mode = ScoreMode::Mixed;
    const int d = weights.config.d_model;
    for (auto& item : mixed.items) {
      item.n_emb_tokens = static_cast<int>(item.tokens.size());
      item.embedding.resize(item.tokens.size() * static_cast<std::size_t>(d));
      for (std::size_t j = 0; j < item.tokens.size(); ++j) {
        const float* row = weights.tok_emb.data() + static_cast<std::size_t>(item.tokens[j]) * d;
        std::copy(row, row + d, item.embedding.begin() + j * d);
      }
      item.tokens.clear();
    }
    const double dev = max_dev(score_ibpc(weights, req), score_mixed(weights, mixed));
    ScoreRequest one_tok = mixed;
    for (auto& item : one_tok.items) {
      item.n_emb_tokens = 1;
      item.embedding.resize(static_cast<std::size_t>(d));
    }
    const auto r = score_mixed(weights, one_tok);
    char buf[160];
    std::snprintf(buf, sizeof(buf), "substitute-embedding dev %.2e <= 1e-6, per-item KV %.1f", dev,
                  r.kv_incremental_per_item);
    criterion(4, "mixed-input equivalence and 1-token KV growth",
              dev <= 1e-6 && r.kv_incremental_per_item == 1.0, buf);
  }
  {  // score_multi_item's single-pass length rule (engine.cpp:195-200)
    Rng rng(7);
    const auto big = seeded_request(rng, 100, 100, 41);  // 4200 > max_seq 4096
    bool threw = false;
    try {
      score_multi_item(weights, big);
    } catch (const Error& e) {
      threw = e.code() == ErrorCode::LengthOverflow;
    }
    const auto chunked = score_multi_item_chunked(weights, big);  // re-batches instead
    criterion(90, "score_multi_item LengthOverflow / chunked accepts", threw &&
              chunked.items.size() == 41, threw ? "threw LengthOverflow" : "no throw");
  }
  {  // text items: build_prompt -> score_by_mode -> score_result_to_json
    ScoreRequest req;
    req.request_id = "text";
    req.mode = ScoreMode::MultiItem;
    const char* docs[] = {"RN, night shift, Boston", "Line cook", "ICU nurse, days"};
    for (int i = 0; i < 3; ++i) {
      const auto parts = build_prompt("Rank jobs for the member.\n", "query: nurse", docs[i]);
      if (req.prefix_tokens.empty()) req.prefix_tokens = parts.prefix_tokens;
      req.items.push_back({std::to_string(10 + i), parts.item_tokens, {}, 0});
    }
    const auto res = score_by_mode(weights, req);
    const auto body = score_result_to_json(res);
    const bool ok = res.items.size() == 3 && body.rfind("{\"flops\":{\"attention\":", 0) == 0 &&
                    body.find("\"request_id\":\"text\"") != std::string::npos &&
                    body.find("\"id\":\"12\"") != std::string::npos;
    criterion(91, "build_prompt items scored and serialised", ok, body.substr(0, 80));
  }
  std::printf(fails ? "acceptance FAILED\n" : "acceptance ok\n");
  return fails ? 1 : 0;
}
