// Host model description: config, weights, init, SRNKWTS1 container.
//
// Mirrors the reference types ModelConfig / ModelWeights (model.hpp:16-67)
// and their invariants (model.cpp:29-92); the container format is the
// reference's SRNKWTS1 (weights_io.hpp:9-14, weights_io.cpp:47-196) so files
// written by either side load in the other.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"

namespace srh {

constexpr int kMinVocabSize = 264;   // tokenizer.hpp:21 (256 bytes + 8 specials)
constexpr int kDefaultMaxSeq = 4096;  // tokenizer.hpp:23
constexpr int kTokenYes = 261, kTokenNo = 262;

struct HeadSpec {
  std::string name;
  int arity = 1;
};

struct ModelConfig {
  int n_layers = 2;
  int d_model = 64;
  int n_heads = 4;
  int d_ff = 256;
  int vocab_size = 300;
  int max_seq = kDefaultMaxSeq;
  int yes_token_id = kTokenYes;
  int no_token_id = kTokenNo;
  std::vector<HeadSpec> head_specs;

  int head_dim() const { return d_model / n_heads; }
  void validate() const;  // SR_SPEC_VIOLATION on a broken invariant
  static ModelConfig default_toy();
  static ModelConfig from_c(const sr_model_config& c);
};

struct LayerWeights {
  std::vector<float> wq, wk, wv, wo;      // [d x d]  (x @ W layout, d_in x d_out)
  std::vector<float> ln1_gain, ln2_gain;  // [d]
  std::vector<float> w_mlp_in;            // [d x ff]
  std::vector<float> w_mlp_out;           // [ff x d]
};

struct TaskHead {
  std::string name;
  int arity = 1;
  std::vector<float> w;  // [d x arity]
  std::vector<float> b;  // [arity]
};

struct ModelWeights {
  ModelConfig config;
  std::string version;
  std::vector<float> tok_emb;  // [V x d]
  std::vector<float> pos_emb;  // [max_seq x d]
  std::vector<LayerWeights> layers;
  std::vector<float> ln_f_gain;  // [d]
  std::vector<float> w_vocab;    // [d x V]
  std::vector<TaskHead> heads;

  void check_shapes() const;
  // Canonical tensor order of the SRNKWTS1 container (weights_io.cpp:47-71).
  std::vector<std::pair<std::string, std::vector<float>*>> tensor_table();
  std::vector<std::pair<std::string, const std::vector<float>*>> tensor_table() const;
  // Allocates every tensor at its config shape (zeros); heads named per spec.
  void allocate();
};

// init_model (model.cpp:94-134). scheme SR_INIT_FAN_IN keeps the reference's
// RNG stream and draw order but scales each tensor's std.
ModelWeights init_model(const ModelConfig& cfg, uint64_t seed, int scheme);

void save_weights(const ModelWeights& w, const std::string& path);
ModelWeights load_weights(const std::string& path);

// splitmix64 stream with FNV-1a named substreams and Box-Muller normals
// (rng.hpp:18-95), bit-reproducible.
class Rng {
 public:
  explicit Rng(uint64_t seed) : state_(seed) {}
  static Rng substream(uint64_t root, const std::string& name);
  uint64_t next_u64();
  double uniform();
  int64_t uniform_int(int64_t lo, int64_t hi);
  double normal(double mean, double stddev);

 private:
  uint64_t state_;
  double spare_ = 0.0;
  bool has_spare_ = false;
};

}  // namespace srh
