// Host model: config invariants, deterministic init, SRNKWTS1 container.
#include "model.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

#include "json_min.hpp"

namespace srh {

// ------------------------------------------------------------------ Rng
Rng Rng::substream(uint64_t root, const std::string& name) {  // rng.hpp:24-31
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : name) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return Rng(root ^ h);
}

uint64_t Rng::next_u64() {  // rng.hpp:33-38 (splitmix64)
  uint64_t z = (state_ += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

double Rng::uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

int64_t Rng::uniform_int(int64_t lo, int64_t hi) {  // rng.hpp:44-47
  const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
  return lo + static_cast<int64_t>(next_u64() % span);
}

double Rng::normal(double mean, double stddev) {  // rng.hpp:52-64 (Box-Muller, cached spare)
  if (has_spare_) {
    has_spare_ = false;
    return mean + stddev * spare_;
  }
  double u1 = uniform(), u2 = uniform();
  while (u1 <= 1e-300) u1 = uniform();
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double theta = 2.0 * 3.141592653589793238462643383279502884 * u2;
  spare_ = r * std::sin(theta);
  has_spare_ = true;
  return mean + stddev * r * std::cos(theta);
}

// --------------------------------------------------------------- config
void ModelConfig::validate() const {  // model.cpp:29-50
  auto bad = [](const std::string& m) { fail(SR_SPEC_VIOLATION, "model config: " + m); };
  if (n_layers < 1 || d_model < 1 || n_heads < 1 || d_ff < 1) bad("all dimensions must be >= 1");
  if (d_model % n_heads != 0) bad("d_model must be divisible by n_heads");
  if (max_seq < 1) bad("max_seq must be >= 1");
  if (yes_token_id == no_token_id) bad("yes and no token ids must differ");
  if (yes_token_id < 0 || yes_token_id >= vocab_size || no_token_id < 0 ||
      no_token_id >= vocab_size)
    bad("yes/no token ids must be < vocab_size");
  if (vocab_size < kMinVocabSize)
    bad("vocab_size must cover bytes plus specials (>= " + std::to_string(kMinVocabSize) + ")");
  for (const auto& h : head_specs)
    if (h.arity < 1) bad("head arity must be >= 1: " + h.name);
}

ModelConfig ModelConfig::default_toy() {  // model.cpp:52-57
  ModelConfig c;
  c.head_specs = {{"click", 1}, {"apply", 1}, {"badfit", 1}, {"shortlist", 1}, {"dismiss", 1}};
  return c;
}

ModelConfig ModelConfig::from_c(const sr_model_config& c) {
  ModelConfig m;
  m.n_layers = c.n_layers;
  m.d_model = c.d_model;
  m.n_heads = c.n_heads;
  m.d_ff = c.d_ff;
  m.vocab_size = c.vocab_size;
  m.max_seq = c.max_seq;
  m.yes_token_id = c.yes_token_id;
  m.no_token_id = c.no_token_id;
  if (c.n_task_heads < 0) fail(SR_SPEC_VIOLATION, "model config: negative head count");
  for (int i = 0; i < c.n_task_heads; ++i) {
    if (c.head_names == nullptr || c.head_names[i] == nullptr || c.head_arity == nullptr)
      fail(SR_SPEC_VIOLATION, "model config: head spec pointers are null");
    m.head_specs.push_back({c.head_names[i], c.head_arity[i]});
  }
  return m;
}

// -------------------------------------------------------------- weights
void ModelWeights::allocate() {
  const size_t d = config.d_model, V = config.vocab_size, S = config.max_seq, F = config.d_ff;
  tok_emb.assign(V * d, 0.f);
  pos_emb.assign(S * d, 0.f);
  layers.assign(config.n_layers, {});
  for (auto& l : layers) {
    l.wq.assign(d * d, 0.f);
    l.wk.assign(d * d, 0.f);
    l.wv.assign(d * d, 0.f);
    l.wo.assign(d * d, 0.f);
    l.ln1_gain.assign(d, 1.f);
    l.ln2_gain.assign(d, 1.f);
    l.w_mlp_in.assign(d * F, 0.f);
    l.w_mlp_out.assign(F * d, 0.f);
  }
  ln_f_gain.assign(d, 1.f);
  w_vocab.assign(d * V, 0.f);
  heads.clear();
  for (const auto& s : config.head_specs) {
    TaskHead h;
    h.name = s.name;
    h.arity = s.arity;
    h.w.assign(d * s.arity, 0.f);
    h.b.assign(s.arity, 0.f);
    heads.push_back(std::move(h));
  }
}

void ModelWeights::check_shapes() const {  // model.cpp:59-92
  const size_t d = config.d_model;
  auto bad = [](const std::string& m) { fail(SR_SPEC_VIOLATION, "model weights: " + m); };
  if (tok_emb.size() != static_cast<size_t>(config.vocab_size) * d) bad("tok_emb shape mismatch");
  if (pos_emb.size() != static_cast<size_t>(config.max_seq) * d) bad("pos_emb shape mismatch");
  if (layers.size() != static_cast<size_t>(config.n_layers)) bad("layer count mismatch");
  for (const auto& l : layers) {
    if (l.wq.size() != d * d || l.wk.size() != d * d || l.wv.size() != d * d ||
        l.wo.size() != d * d || l.ln1_gain.size() != d || l.ln2_gain.size() != d ||
        l.w_mlp_in.size() != d * static_cast<size_t>(config.d_ff) ||
        l.w_mlp_out.size() != static_cast<size_t>(config.d_ff) * d)
      bad("layer tensor shape mismatch");
  }
  if (ln_f_gain.size() != d) bad("ln_f shape mismatch");
  if (w_vocab.size() != d * static_cast<size_t>(config.vocab_size)) bad("w_vocab shape mismatch");
  if (heads.size() != config.head_specs.size()) bad("head count mismatch");
  for (size_t i = 0; i < heads.size(); ++i) {
    const size_t a = config.head_specs[i].arity;
    if (heads[i].w.size() != d * a || heads[i].b.size() != a)
      bad("head tensor shape mismatch: " + heads[i].name);
  }
}

template <typename W, typename Ref>
static std::vector<Ref> table_of(W& w) {  // weights_io.cpp:47-71
  std::vector<Ref> refs;
  refs.push_back({"tok_emb", &w.tok_emb});
  refs.push_back({"pos_emb", &w.pos_emb});
  for (size_t i = 0; i < w.layers.size(); ++i) {
    auto& l = w.layers[i];
    const std::string p = "layers." + std::to_string(i) + ".";
    refs.push_back({p + "wq", &l.wq});
    refs.push_back({p + "wk", &l.wk});
    refs.push_back({p + "wv", &l.wv});
    refs.push_back({p + "wo", &l.wo});
    refs.push_back({p + "ln1_gain", &l.ln1_gain});
    refs.push_back({p + "ln2_gain", &l.ln2_gain});
    refs.push_back({p + "w_mlp_in", &l.w_mlp_in});
    refs.push_back({p + "w_mlp_out", &l.w_mlp_out});
  }
  refs.push_back({"ln_f_gain", &w.ln_f_gain});
  refs.push_back({"w_vocab", &w.w_vocab});
  for (auto& h : w.heads) {
    refs.push_back({"heads." + h.name + ".w", &h.w});
    refs.push_back({"heads." + h.name + ".b", &h.b});
  }
  return refs;
}

std::vector<std::pair<std::string, std::vector<float>*>> ModelWeights::tensor_table() {
  return table_of<ModelWeights, std::pair<std::string, std::vector<float>*>>(*this);
}
std::vector<std::pair<std::string, const std::vector<float>*>> ModelWeights::tensor_table() const {
  return table_of<const ModelWeights, std::pair<std::string, const std::vector<float>*>>(*this);
}

// ----------------------------------------------------------------- init
namespace {
void fill_normal(Rng& rng, std::vector<float>& t, size_t n, double stddev) {
  t.resize(n);
  for (auto& v : t) v = static_cast<float>(std::clamp(rng.normal(0.0, stddev), -1.0, 1.0));
}
}  // namespace

ModelWeights init_model(const ModelConfig& cfg, uint64_t seed, int scheme) {
  cfg.validate();
  if (scheme != SR_INIT_REFERENCE && scheme != SR_INIT_FAN_IN)
    fail(SR_PARAMETER, "unknown init scheme " + std::to_string(scheme));
  Rng rng = Rng::substream(seed, "init");
  ModelWeights w;
  w.config = cfg;
  char buf[40];
  std::snprintf(buf, sizeof(buf), scheme == SR_INIT_REFERENCE ? "toy-%016llx" : "fanin-%016llx",
                static_cast<unsigned long long>(seed));
  w.version = buf;

  // kInitStd = 0.08f (model.cpp:18) promoted to double at the call.
  const double ref_std = static_cast<double>(0.08f);
  const bool fan = scheme == SR_INIT_FAN_IN;
  const size_t d = cfg.d_model, F = cfg.d_ff;
  const double resid = std::sqrt(2.0 * cfg.n_layers);
  const double s_d = fan ? 1.0 / std::sqrt(static_cast<double>(d)) : ref_std;
  const double s_o = fan ? 1.0 / std::sqrt(static_cast<double>(d)) / resid : ref_std;
  const double s_ff = fan ? 1.0 / std::sqrt(static_cast<double>(F)) / resid : ref_std;

  fill_normal(rng, w.tok_emb, static_cast<size_t>(cfg.vocab_size) * d, ref_std);
  fill_normal(rng, w.pos_emb, static_cast<size_t>(cfg.max_seq) * d, ref_std);
  w.layers.resize(cfg.n_layers);
  for (auto& l : w.layers) {
    fill_normal(rng, l.wq, d * d, s_d);
    fill_normal(rng, l.wk, d * d, s_d);
    fill_normal(rng, l.wv, d * d, s_d);
    fill_normal(rng, l.wo, d * d, s_o);
    l.ln1_gain.assign(d, 1.0f);
    l.ln2_gain.assign(d, 1.0f);
    fill_normal(rng, l.w_mlp_in, d * F, s_d);
    fill_normal(rng, l.w_mlp_out, F * d, s_ff);
  }
  w.ln_f_gain.assign(d, 1.0f);
  fill_normal(rng, w.w_vocab, d * static_cast<size_t>(cfg.vocab_size), s_d);
  for (const auto& spec : cfg.head_specs) {
    TaskHead h;
    h.name = spec.name;
    h.arity = spec.arity;
    fill_normal(rng, h.w, d * static_cast<size_t>(spec.arity), s_d);
    h.b.assign(spec.arity, 0.0f);
    w.heads.push_back(std::move(h));
  }
  return w;
}

// ------------------------------------------------------------ container
namespace {
constexpr char kMagic[8] = {'S', 'R', 'N', 'K', 'W', 'T', 'S', '1'};
constexpr uint32_t kFormatVersion = 1;

// Manifest text identical to nlohmann::json::dump() of the reference's
// manifest (weights_io.cpp:56-66,110-117): object keys sorted, compact.
std::string manifest_text(const ModelWeights& w) {
  const auto& c = w.config;
  std::ostringstream o;
  o << "{\"config\":{\"d_ff\":" << c.d_ff << ",\"d_model\":" << c.d_model << ",\"head_specs\":[";
  for (size_t i = 0; i < c.head_specs.size(); ++i) {
    if (i) o << ',';
    o << "{\"arity\":" << c.head_specs[i].arity << ",\"name\":" << json::quote(c.head_specs[i].name)
      << '}';
  }
  o << "],\"max_seq\":" << c.max_seq << ",\"n_heads\":" << c.n_heads
    << ",\"n_layers\":" << c.n_layers << ",\"no_token_id\":" << c.no_token_id
    << ",\"vocab_size\":" << c.vocab_size << ",\"yes_token_id\":" << c.yes_token_id << "}";
  o << ",\"model_version\":" << json::quote(w.version) << ",\"tensors\":[";
  uint64_t offset = 0;
  bool first = true;
  for (const auto& [name, t] : w.tensor_table()) {
    if (!first) o << ',';
    first = false;
    o << "{\"name\":" << json::quote(name) << ",\"offset\":" << offset << ",\"shape\":[" << t->size()
      << "]}";
    offset += t->size() * sizeof(float);
  }
  o << "]}";
  return o.str();
}
}  // namespace

void save_weights(const ModelWeights& w, const std::string& path) {  // weights_io.cpp:104-135
  w.check_shapes();
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) fail(SR_IO, "cannot open for write: " + path);
  const std::string m = manifest_text(w);
  out.write(kMagic, sizeof(kMagic));
  const uint32_t ver = kFormatVersion;
  out.write(reinterpret_cast<const char*>(&ver), sizeof(ver));
  const uint64_t len = m.size();
  out.write(reinterpret_cast<const char*>(&len), sizeof(len));
  out.write(m.data(), static_cast<std::streamsize>(m.size()));
  for (const auto& [name, t] : w.tensor_table())
    out.write(reinterpret_cast<const char*>(t->data()),
              static_cast<std::streamsize>(t->size() * sizeof(float)));
  if (!out) fail(SR_IO, "write failed: " + path);
}

ModelWeights load_weights(const std::string& path) {  // weights_io.cpp:137-196
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(SR_IO, "cannot open: " + path);
  char magic[8];
  in.read(magic, sizeof(magic));
  if (!in || std::memcmp(magic, kMagic, sizeof(kMagic)) != 0)
    fail(SR_IO, "bad magic in weight file: " + path);
  uint32_t ver = 0;
  in.read(reinterpret_cast<char*>(&ver), sizeof(ver));
  if (!in || ver != kFormatVersion) fail(SR_IO, "unsupported weight format version");
  uint64_t mlen = 0;
  in.read(reinterpret_cast<char*>(&mlen), sizeof(mlen));
  if (!in || mlen > (1ull << 32)) fail(SR_IO, "truncated manifest: " + path);
  std::string text(mlen, '\0');
  in.read(text.data(), static_cast<std::streamsize>(mlen));
  if (!in) fail(SR_IO, "truncated manifest: " + path);
  json::Value man;
  try {
    man = json::parse(text);
  } catch (const Error& e) {
    fail(SR_IO, std::string("manifest parse error: ") + e.what());
  }
  ModelWeights w;
  const auto& jc = man.at("config");
  auto& c = w.config;
  c.n_layers = static_cast<int>(jc.at("n_layers").as_int());
  c.d_model = static_cast<int>(jc.at("d_model").as_int());
  c.n_heads = static_cast<int>(jc.at("n_heads").as_int());
  c.d_ff = static_cast<int>(jc.at("d_ff").as_int());
  c.vocab_size = static_cast<int>(jc.at("vocab_size").as_int());
  c.max_seq = static_cast<int>(jc.at("max_seq").as_int());
  c.yes_token_id = static_cast<int>(jc.at("yes_token_id").as_int());
  c.no_token_id = static_cast<int>(jc.at("no_token_id").as_int());
  c.head_specs.clear();
  for (const auto& h : jc.at("head_specs").arr)
    c.head_specs.push_back({h.at("name").as_str(), static_cast<int>(h.at("arity").as_int())});
  c.validate();
  w.version = man.at("model_version").as_str();
  w.layers.resize(c.n_layers);
  for (const auto& s : c.head_specs) w.heads.push_back({s.name, s.arity, {}, {}});
  auto refs = w.tensor_table();
  size_t next = 0;
  for (const auto& e : man.at("tensors").arr) {
    const std::string name = e.at("name").as_str();
    if (next >= refs.size() || refs[next].first != name)
      fail(SR_IO, "unexpected tensor in manifest: " + name);
    uint64_t n = 1;
    for (const auto& dim : e.at("shape").arr) n *= dim.as_uint();
    auto* t = refs[next].second;
    t->resize(n);
    in.read(reinterpret_cast<char*>(t->data()), static_cast<std::streamsize>(n * sizeof(float)));
    if (!in) fail(SR_IO, "truncated tensor data: " + name);
    ++next;
  }
  if (next != refs.size()) fail(SR_IO, "weight file missing tensors");
  w.check_shapes();
  return w;
}

// --------------------------------------------------------------- json
namespace json {

namespace {
struct Parser {
  const std::string& s;
  size_t i = 0;
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r')) ++i;
  }
  [[noreturn]] void err(const char* m) { fail(SR_IO, std::string("json: ") + m + " at " + std::to_string(i)); }
  char peek() {
    ws();
    if (i >= s.size()) err("unexpected end");
    return s[i];
  }
  void expect(char c) {
    if (peek() != c) err("unexpected character");
    ++i;
  }
  std::string str() {
    expect('"');
    std::string out;
    while (true) {
      if (i >= s.size()) err("unterminated string");
      char c = s[i++];
      if (c == '"') break;
      if (c == '\\') {
        if (i >= s.size()) err("bad escape");
        char e = s[i++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (i + 4 > s.size()) err("bad unicode escape");
            unsigned cp = std::stoul(s.substr(i, 4), nullptr, 16);
            i += 4;
            if (cp < 0x80) {
              out += static_cast<char>(cp);
            } else if (cp < 0x800) {
              out += static_cast<char>(0xC0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              out += static_cast<char>(0xE0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default: err("bad escape");
        }
      } else {
        out += c;
      }
    }
    return out;
  }
  Value value() {
    Value v;
    char c = peek();
    if (c == '{') {
      ++i;
      v.kind = Value::Object;
      if (peek() == '}') {
        ++i;
        return v;
      }
      while (true) {
        std::string k = str();
        expect(':');
        v.obj.emplace_back(std::move(k), value());
        char n = peek();
        ++i;
        if (n == '}') break;
        if (n != ',') err("expected , or }");
      }
    } else if (c == '[') {
      ++i;
      v.kind = Value::Array;
      if (peek() == ']') {
        ++i;
        return v;
      }
      while (true) {
        v.arr.push_back(value());
        char n = peek();
        ++i;
        if (n == ']') break;
        if (n != ',') err("expected , or ]");
      }
    } else if (c == '"') {
      v.kind = Value::String;
      v.text = str();
    } else if (s.compare(i, 4, "true") == 0) {
      v.kind = Value::Bool;
      v.b = true;
      i += 4;
    } else if (s.compare(i, 5, "false") == 0) {
      v.kind = Value::Bool;
      i += 5;
    } else if (s.compare(i, 4, "null") == 0) {
      i += 4;
    } else {
      size_t j = i;
      while (j < s.size() && (std::isdigit(static_cast<unsigned char>(s[j])) || s[j] == '-' ||
                              s[j] == '+' || s[j] == '.' || s[j] == 'e' || s[j] == 'E'))
        ++j;
      if (j == i) err("unexpected token");
      v.kind = Value::Number;
      v.text = s.substr(i, j - i);
      i = j;
    }
    return v;
  }
};
}  // namespace

Value parse(const std::string& s) {
  Parser p{s};
  Value v = p.value();
  p.ws();
  if (p.i != s.size()) p.err("trailing characters");
  return v;
}

std::string quote(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    switch (c) {
      case '"': o += "\\\""; break;
      case '\\': o += "\\\\"; break;
      case '\b': o += "\\b"; break;
      case '\f': o += "\\f"; break;
      case '\n': o += "\\n"; break;
      case '\r': o += "\\r"; break;
      case '\t': o += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof(b), "\\u%04x", c);
          o += b;
        } else {
          o += static_cast<char>(c);
        }
    }
  }
  return o + "\"";
}

}  // namespace json

}  // namespace srh
