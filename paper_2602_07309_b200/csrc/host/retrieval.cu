// Device-resident corpus + exhaustive filtered top-K.
// Host half of kernels/retrieval.cu; mirrors exhaustive_topk's contract
// (retrieval.hpp:60-70, retrieval.cpp:134-173): precondition order, error
// codes, (score desc, doc_id asc) order, min(k, candidates) results.
#include <cmath>
#include <cstring>

#include "engine.hpp"
#include "retrieval.hpp"

namespace srh {

Corpus::Corpus(const float* emb, const float* feat, const int64_t* ids, long long n, int d_emb,
               int n_feat, int device)
    : device_(device), n_(n), d_(d_emb), f_(n_feat) {
  if (n < 0 || d_emb < 1 || n_feat < 0) fail(SR_PARAMETER, "corpus dimensions must be positive");
  if (n > INT32_MAX) fail(SR_PARAMETER, "corpus larger than 2^31 docs per device");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(SR_CUDA, "no CUDA device: the retrieval scan has no CPU fallback");
  if (device < 0 || device >= ndev) fail(SR_PARAMETER, "device index out of range");
  SR_CUDA_CHECK(cudaSetDevice(device));
  SR_CUDA_CHECK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  const size_t nn = static_cast<size_t>(std::max<long long>(n, 1));
  SR_CUDA_CHECK(cudaMalloc(&emb_, nn * d_ * sizeof(float)));
  SR_CUDA_CHECK(cudaMalloc(&feat_, nn * std::max(f_, 1) * sizeof(float)));
  SR_CUDA_CHECK(cudaMalloc(&ids_, nn * sizeof(int64_t)));
  SR_CUDA_CHECK(cudaMalloc(&keep_, nn));
  SR_CUDA_CHECK(cudaMalloc(&vec_, 4 * sizeof(double) * (d_ + f_ + 2)));
  SR_CUDA_CHECK(cudaMalloc(&counters_, 2 * sizeof(int32_t)));
  if (n > 0) {
    SR_CUDA_CHECK(cudaMemcpyAsync(emb_, emb, static_cast<size_t>(n) * d_ * sizeof(float),
                                  cudaMemcpyHostToDevice, stream_));
    if (f_ > 0)
      SR_CUDA_CHECK(cudaMemcpyAsync(feat_, feat, static_cast<size_t>(n) * f_ * sizeof(float),
                                    cudaMemcpyHostToDevice, stream_));
    SR_CUDA_CHECK(cudaMemcpyAsync(ids_, ids, static_cast<size_t>(n) * sizeof(int64_t),
                                  cudaMemcpyHostToDevice, stream_));
  }
  // |f_i| bounds for the fp32 pre-pass error bound
  fmax_.assign(f_, 0.0);
  for (long long i = 0; i < n; ++i)
    for (int j = 0; j < f_; ++j)
      fmax_[j] = std::max(fmax_[j], std::fabs(static_cast<double>(feat[i * f_ + j])));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  grid_ = 4 * sms;
  cand_cap_ = grid_ * 1024;
  SR_CUDA_CHECK(cudaMalloc(&cand_, static_cast<size_t>(cand_cap_) * sizeof(int32_t)));
  SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
}

Corpus::~Corpus() {
  cudaSetDevice(device_);
  for (void* p : {static_cast<void*>(emb_), static_cast<void*>(feat_), static_cast<void*>(ids_),
                  static_cast<void*>(keep_), static_cast<void*>(vec_),
                  static_cast<void*>(counters_), static_cast<void*>(cand_)})
    if (p) cudaFree(p);
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  if (stream_) cudaStreamDestroy(stream_);
}

long long Corpus::prepare(const float* query, int d_query, double w0, const double* w, int n_w,
                          const uint8_t* keep, int k, srk::RetrievalScan& a) {
  if (k < 1) fail(SR_SPEC_VIOLATION, "top-K requires K >= 1");
  long long n_keep = n_;
  if (keep != nullptr) {
    n_keep = 0;
    for (long long i = 0; i < n_; ++i) n_keep += keep[i] != 0;
  }
  if (n_keep == 0) return 0;  // nothing scored: no per-candidate checks run
  // rar_score (retrieval.cpp:60-64) checks the weights, then cosine (:44-56)
  if (n_w != f_) fail(SR_ALIGNMENT, "feature count does not match RAR weight count");
  if (d_query != d_ || d_query == 0) fail(SR_ALIGNMENT, "cosine: dimension mismatch");
  double na = 0.0;
  for (int i = 0; i < d_; ++i) na += static_cast<double>(query[i]) * query[i];
  if (na == 0.0) fail(SR_DEGENERATE_INPUT, "cosine of a zero vector");
  // staging: [q32 (d) | w32 (f)] as float, [qd (d) | wd (f)] as double
  h32_.ensure(static_cast<size_t>(d_ + f_ + 1));
  h64_.ensure(static_cast<size_t>(d_ + f_ + 1));
  float* f32 = h32_.ptr;
  double* f64 = h64_.ptr;
  for (int i = 0; i < d_; ++i) {
    f32[i] = query[i];
    f64[i] = static_cast<double>(query[i]);
  }
  double wsum = std::fabs(w0);
  for (int j = 0; j < f_; ++j) {
    f32[d_ + j] = static_cast<float>(w[j]);
    f64[d_ + j] = w[j];
    wsum += std::fabs(w[j]) * fmax_[j];
  }
  float* v32 = reinterpret_cast<float*>(vec_);
  double* v64 = vec_ + (d_ + f_ + 2);
  SR_CUDA_CHECK(cudaMemcpyAsync(v32, f32, (d_ + f_ + 1) * sizeof(float), cudaMemcpyHostToDevice,
                                stream_));
  SR_CUDA_CHECK(cudaMemcpyAsync(v64, f64, (d_ + f_ + 1) * sizeof(double), cudaMemcpyHostToDevice,
                                stream_));
  if (keep != nullptr)
    SR_CUDA_CHECK(cudaMemcpyAsync(keep_, keep, static_cast<size_t>(n_), cudaMemcpyHostToDevice,
                                  stream_));
  // Rigorous bound on |s32 - s64|: fp32 dot/norm accumulation
  // over D terms (gamma_D), sqrt/div/scale roundings, fp32 weights/features.
  const double u = std::ldexp(1.0, -24);
  const double gD = d_ * u / (1.0 - d_ * u);
  const double eps = 2.0 * (std::fabs(w0) * (3.0 * gD + 8.0 * u) + (f_ + 3) * u * wsum) + 1e-12;
  a.emb = emb_;
  a.feat = feat_;
  a.ids = ids_;
  a.keep = keep != nullptr ? keep_ : nullptr;
  a.q32 = v32;
  a.w32 = v32 + d_;
  a.qd = v64;
  a.wd = v64 + d_;
  a.w0 = w0;
  a.q_norm = std::sqrt(na);
  a.eps2 = static_cast<float>(2.0 * eps);
  a.n = n_;
  a.D = d_;
  a.F = f_;
  a.k = k;
  return n_keep;
}

int Corpus::topk(const float* query, int d_query, double w0, const double* w, int n_w,
                 const uint8_t* keep, int k, srk::TopkEntry* dev_out) {
  SR_CUDA_CHECK(cudaSetDevice(device_));
  srk::RetrievalScan a;
  const long long n_keep = prepare(query, d_query, w0, w, n_w, keep, k, a);
  if (n_keep == 0) return 0;
  if (k > kScanMaxK) {
    // Large K (the reference allows K up to and past the corpus size): every
    // doc rescored in double, then the multi-level bitonic selection of the
    // exact top K (K <= 2048) or, past that, a full stable sort.
    SR_CUDA_CHECK(cudaMemsetAsync(counters_, 0, 2 * sizeof(int32_t), stream_));
    entries_.ensure(static_cast<size_t>(n_));
    SR_CUDA_CHECK(srk::retrieval_refine(a, nullptr, n_, entries_.ptr, counters_, stream_));
    hcnt_.ensure(2);
    int32_t* cnt = hcnt_.ptr;
    SR_CUDA_CHECK(cudaMemcpyAsync(cnt, counters_, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                  stream_));
    SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
    if (cnt[1] & 1) fail(SR_DEGENERATE_INPUT, "cosine of a zero vector");
    if (k <= srk::kTopkSelectMaxK) {
      select_.ensure(srk::topk_select_scratch(n_, k));
      SR_CUDA_CHECK(srk::topk_select(entries_.ptr, n_, k, select_.ptr, dev_out, stream_));
    } else {
      const size_t bytes = srk::retrieval_sort_scratch(n_);
      sort_.ensure(bytes);
      SR_CUDA_CHECK(
          srk::retrieval_sort_topk(entries_.ptr, n_, k, sort_.ptr, bytes, dev_out, stream_));
    }
    last_candidates_ = n_;
    return static_cast<int>(std::min<long long>(k, n_keep));
  }
  if (!ev_[0]) {
    SR_CUDA_CHECK(cudaEventCreate(&ev_[0]));
    SR_CUDA_CHECK(cudaEventCreate(&ev_[1]));
  }
  SR_CUDA_CHECK(cudaEventRecord(ev_[0], stream_));
  SR_CUDA_CHECK(srk::retrieval_scan(a, cand_, cand_cap_, counters_, grid_, stream_));
  SR_CUDA_CHECK(cudaEventRecord(ev_[1], stream_));
  hcnt_.ensure(2);
  int32_t* cnt = hcnt_.ptr;
  SR_CUDA_CHECK(cudaMemcpyAsync(cnt, counters_, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                stream_));
  SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
  SR_CUDA_CHECK(cudaEventElapsedTime(&last_scan_ms_, ev_[0], ev_[1]));
  if (cnt[1] & 1) fail(SR_DEGENERATE_INPUT, "cosine of a zero vector");
  const bool exact_all = (cnt[1] & 2) != 0;  // near-tie overflow: rescore every doc
  const long long m = exact_all ? n_ : cnt[0];
  entries_.ensure(static_cast<size_t>(std::max<long long>(m, 1)));
  select_.ensure(srk::topk_select_scratch(m, k));
  SR_CUDA_CHECK(srk::retrieval_refine(a, exact_all ? nullptr : cand_, m, entries_.ptr, counters_,
                                      stream_));
  SR_CUDA_CHECK(srk::topk_select(entries_.ptr, m, k, select_.ptr, dev_out, stream_));
  last_candidates_ = m;
  return static_cast<int>(std::min<long long>(k, n_keep));
}

int Corpus::topk_host(const float* query, int d_query, double w0, const double* w, int n_w,
                      const uint8_t* keep, int k, int64_t* ids_out, double* scores_out) {
  if (k < 1) fail(SR_SPEC_VIOLATION, "top-K requires K >= 1");
  out_.ensure(static_cast<size_t>(std::max(k, 1)));
  const int n = topk(query, d_query, w0, w, n_w, keep, k, out_.ptr);
  if (n == 0) return 0;
  hout_.ensure(static_cast<size_t>(n));
  srk::TopkEntry* h = hout_.ptr;
  SR_CUDA_CHECK(cudaMemcpyAsync(h, out_.ptr, sizeof(srk::TopkEntry) * n, cudaMemcpyDeviceToHost,
                                stream_));
  SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
  for (int j = 0; j < n; ++j) {
    if (ids_out) ids_out[j] = h[j].id;
    if (scores_out) scores_out[j] = h[j].score;
  }
  return n;
}

int Corpus::topk_sharded(Comm* c, const float* query, int d_query, double w0, const double* w,
                         int n_w, const uint8_t* keep, int k, int64_t* ids_out,
                         double* scores_out) {
  if (c == nullptr) return topk_host(query, d_query, w0, w, n_w, keep, k, ids_out, scores_out);
  if (k < 1) fail(SR_SPEC_VIOLATION, "top-K requires K >= 1");
  if (static_cast<long>(c->nranks) * k > 4096) fail(SR_PARAMETER, "nranks * k must be <= 4096");
  SR_CUDA_CHECK(cudaSetDevice(device_));
  out_.ensure(static_cast<size_t>(k));
  gathered_.ensure(static_cast<size_t>(c->nranks) * k);
  merged_.ensure(static_cast<size_t>(k));
  // every rank contributes exactly k entries (sentinel-padded) so the
  // all-gather has one shape; sentinels sort last in the merge
  const int n = topk(query, d_query, w0, w, n_w, keep, k, out_.ptr);
  if (n < k) {
    std::vector<srk::TopkEntry> s(k - n);
    for (auto& e : s) {
      e.score = -INFINITY;
      e.id = INT64_MAX;
      e.index = INT32_MAX;
      e.pad = 0;
    }
    SR_CUDA_CHECK(cudaMemcpyAsync(out_.ptr + n, s.data(), sizeof(srk::TopkEntry) * (k - n),
                                  cudaMemcpyHostToDevice, stream_));
  }
  nccl_allgather_bytes(c, out_.ptr, gathered_.ptr, sizeof(srk::TopkEntry) * k, stream_);
  SR_CUDA_CHECK(srk::topk_merge(gathered_.ptr, c->nranks * k, k, merged_.ptr, stream_));
  std::vector<srk::TopkEntry> h(k);
  SR_CUDA_CHECK(cudaMemcpyAsync(h.data(), merged_.ptr, sizeof(srk::TopkEntry) * k,
                                cudaMemcpyDeviceToHost, stream_));
  SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
  int m = 0;
  for (; m < k && h[m].index != INT32_MAX; ++m) {  // sentinel by index: any int64 is a valid doc id
    if (ids_out) ids_out[m] = h[m].id;
    if (scores_out) scores_out[m] = h[m].score;
  }
  return m;
}

}  // namespace srh
