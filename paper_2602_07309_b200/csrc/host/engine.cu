// Device engine implementation: weight conversion, workspace, the packed
// forward (one launch sequence per request batch), CUDA-graph plans, NCCL.
//
// Forward for a packed batch (model.cpp:149-220 restated for B200):
//   embed+LN1      x = emb + pos (fp32 residual), xn = bf16 LN1(x)
//   per layer l:   qkv = xn Wqkv^T                 tcgen05 GEMM, bf16 out
//                  xn  = attention(qkv, spans)     segment-masked, bf16 out
//                  x  += xn Wo^T                   tcgen05 GEMM, fp32 residual epilogue
//                  xn  = LN2(x)
//                  h   = gelu(xn Win^T)            tcgen05 GEMM, GELU epilogue
//                  x  += h Wout^T                  tcgen05 GEMM, fp32 residual epilogue
//                  xn  = LN1_{l+1}(x)              (skipped after the last layer)
//   score head on the items' last rows (final LN fused), then top-k.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "engine.hpp"

namespace srh {

namespace {

template <typename T>
T* upload(const std::vector<T>& v, std::vector<void*>& allocs) {
  T* p = nullptr;
  SR_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(v.size(), 1) * sizeof(T)));
  allocs.push_back(p);
  if (!v.empty()) {
    SR_CUDA_CHECK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    SR_CUDA_CHECK(cudaDeviceSynchronize());  // pageable copies may still be in flight
  }
  return p;
}

void make_weight_map(CUtensorMap* m, const void* w, int rows, int cols) {
  SR_CUDA_CHECK(srk::make_tmap_bf16_2d(m, w, rows, cols, srk::gemm_b_box_rows(rows), 64));
}

}  // namespace

Engine::Engine(const ModelWeights& w, int device) : cfg_(w.config), device_(device) {
  w.check_shapes();
  cfg_.validate();
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(SR_CUDA, "no CUDA device: the B200 ranker has no CPU fallback");
  if (device < 0 || device >= ndev) fail(SR_PARAMETER, "device index out of range");
  SR_CUDA_CHECK(cudaSetDevice(device));
  cudaDeviceProp prop;
  SR_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    fail(SR_CUDA, std::string("requires an sm_100 (Blackwell) device, found ") + prop.name);
  const int d = cfg_.d_model, F = cfg_.d_ff;
  if (d % 64 != 0 || F % 64 != 0)
    fail(SR_SPEC_VIOLATION, "d_model and d_ff must be multiples of 64 on the tcgen05 path");
  const int hd = cfg_.head_dim();
  if (hd != 16 && hd != 32 && hd != 64 && hd != 128)
    fail(SR_SPEC_VIOLATION, "head_dim must be one of 16/32/64/128");
  SR_CUDA_CHECK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  SR_CUDA_CHECK(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
  SR_CUDA_CHECK(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  SR_CUDA_CHECK(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
  // Opt-in (SRK_FOLD_LN=1): LN folded into the projections when every GEMM
  // takes the pair kernel. Measured on B200 at C2 it breaks even with the
  // separate LayerNorm kernel (the residual epilogue's extra x traffic slows
  // the main loop as much as the LN launches cost), so it is off by default.
  {
    const char* v = std::getenv("SRK_FOLD_LN");
    const bool allow = v != nullptr && std::atoi(v) != 0;
    fold_ln_ = allow && srk::gemm_use_pair(d) && srk::gemm_use_pair(3 * d) &&
               srk::gemm_use_pair(F) && d % 128 == 0 && d / 128 <= 16;
    const char* sv = std::getenv("SRK_SERPENTINE");
    serpentine_ = sv == nullptr || std::atoi(sv) != 0;
    // Opt-in (SRK_LN_AFTER=1): the next LayerNorm overlapped with each
    // residual GEMM (epilogue 7 + layer_norm_after on a side stream). Measured
    // slower at C2 (9.84 vs 8.97 ms per query): the GEMM is at the HBM ridge
    // and the concurrent LayerNorm slows both.
    // LPT order of the attention work items (SRK_ATTN_LPT=0: head-major)
    const char* av = std::getenv("SRK_ATTN_LPT");
    attn_lpt_ = av == nullptr || std::atoi(av) != 0;
    // a request with the plan's last layout re-uploads only its token ids and
    // doc ids (SRK_LAYOUT_REUSE=0: full repack and upload every call)
    const char* rv = std::getenv("SRK_LAYOUT_REUSE");
    layout_reuse_ = rv == nullptr || std::atoi(rv) != 0;
    const char* lv = std::getenv("SRK_LN_AFTER");
    ln_after_ = !fold_ln_ && lv != nullptr && std::atoi(lv) != 0 && srk::gemm_use_pair(d) &&
                d % 4 == 0 && d <= 2048;
  }

  tok_emb_ = upload(w.tok_emb, allocs_);
  pos_emb_ = upload(w.pos_emb, allocs_);
  ln_f_ = upload(w.ln_f_gain, allocs_);

  // fp32 [K x N] staging -> bf16 [N x K] (K-major B operand) on the device.
  float* stage = nullptr;
  const size_t stage_elems = static_cast<size_t>(std::max(d, F)) * std::max(d, F);
  SR_CUDA_CHECK(cudaMalloc(&stage, stage_elems * sizeof(float)));
  auto conv = [&](const std::vector<float>& src, __nv_bfloat16* dst, int K, int N,
                  const float* scale_k) {
    // Same-stream copy: a pageable cudaMemcpy may return before its DMA lands,
    // and stream_ is non-blocking w.r.t. the legacy stream.
    SR_CUDA_CHECK(cudaMemcpyAsync(stage, src.data(), src.size() * sizeof(float),
                                  cudaMemcpyHostToDevice, stream_));
    SR_CUDA_CHECK(srk::transpose_to_bf16(stage, dst, K, N, stream_, scale_k));
    SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
  };
  layers_.resize(cfg_.n_layers);
  for (int l = 0; l < cfg_.n_layers; ++l) {
    const auto& lw = w.layers[l];
    auto& L = layers_[l];
    auto alloc_bf16 = [&](size_t n) {
      __nv_bfloat16* p = nullptr;
      SR_CUDA_CHECK(cudaMalloc(&p, n * sizeof(__nv_bfloat16)));
      allocs_.push_back(p);
      return p;
    };
    L.wqkv = alloc_bf16(static_cast<size_t>(3) * d * d);
    L.wo = alloc_bf16(static_cast<size_t>(d) * d);
    L.win = alloc_bf16(static_cast<size_t>(F) * d);
    L.wout = alloc_bf16(static_cast<size_t>(d) * F);
    L.ln1 = upload(lw.ln1_gain, allocs_);
    L.ln2 = upload(lw.ln2_gain, allocs_);
    // Folded LN: the gains scale the K rows of the following projection.
    const float* g1 = fold_ln_ ? L.ln1 : nullptr;
    const float* g2 = fold_ln_ ? L.ln2 : nullptr;
    conv(lw.wq, L.wqkv, d, d, g1);
    conv(lw.wk, L.wqkv + static_cast<size_t>(d) * d, d, d, g1);
    conv(lw.wv, L.wqkv + static_cast<size_t>(2) * d * d, d, d, g1);
    conv(lw.wo, L.wo, d, d, nullptr);
    conv(lw.w_mlp_in, L.win, d, F, g2);
    conv(lw.w_mlp_out, L.wout, F, d, nullptr);
    if (fold_ln_) {
      SR_CUDA_CHECK(cudaMalloc(&L.cs_qkv, sizeof(float) * 3 * d));
      allocs_.push_back(L.cs_qkv);
      SR_CUDA_CHECK(cudaMalloc(&L.cs_in, sizeof(float) * F));
      allocs_.push_back(L.cs_in);
      SR_CUDA_CHECK(srk::bf16_row_sums(L.wqkv, 3 * d, d, L.cs_qkv, stream_));
      SR_CUDA_CHECK(srk::bf16_row_sums(L.win, F, d, L.cs_in, stream_));
      SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
    }
    make_weight_map(&L.tm_qkv, L.wqkv, 3 * d, d);
    make_weight_map(&L.tm_o, L.wo, d, d);
    make_weight_map(&L.tm_in, L.win, F, d);
    make_weight_map(&L.tm_out, L.wout, d, F);
  }
  cudaFree(stage);

  // Score-head columns: [w_vocab[:,yes], w_vocab[:,no], head columns...].
  const int V = cfg_.vocab_size;
  std::vector<float> cols, bias;
  std::vector<int32_t> tcol, tar;
  auto add_col = [&](auto get, float b) {
    for (int j = 0; j < d; ++j) cols.push_back(get(j));
    bias.push_back(b);
  };
  add_col([&](int j) { return w.w_vocab[static_cast<size_t>(j) * V + cfg_.yes_token_id]; }, 0.f);
  add_col([&](int j) { return w.w_vocab[static_cast<size_t>(j) * V + cfg_.no_token_id]; }, 0.f);
  yes_col_ = 0;
  no_col_ = 1;
  for (const auto& h : w.heads) {
    tcol.push_back(static_cast<int32_t>(bias.size()));
    tar.push_back(h.arity);
    for (int a = 0; a < h.arity; ++a)
      add_col([&](int j) { return h.w[static_cast<size_t>(j) * h.arity + a]; }, h.b[a]);
  }
  n_cols_ = static_cast<int>(bias.size());
  head_w_ = upload(cols, allocs_);
  head_b_ = upload(bias, allocs_);
  task_col_ = upload(tcol, allocs_);
  task_arity_ = upload(tar, allocs_);
  SR_CUDA_CHECK(cudaDeviceSynchronize());
}

Engine::~Engine() {
  cache_.clear();
  cudaSetDevice(device_);
  for (void* p : allocs_) cudaFree(p);
  if (stream_) cudaStreamDestroy(stream_);
  if (side_) cudaStreamDestroy(side_);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
}

Plan::~Plan() {
  if (graph) cudaGraphExecDestroy(graph);
}

void Engine::set_postprocess(const double* lo, const double* hi, const double* value,
                             int n_blocks, const int32_t* blend_task, const double* blend_w,
                             int n_blend) {
  if (n_blocks < 0 || n_blend < 0) fail(SR_PARAMETER, "negative post-processing size");
  // handle_search always calibrates the relevance before blending, and
  // calibrate() rejects an unfitted head (calibration.cpp:65-68).
  if (n_blend > 0 && n_blocks == 0) fail(SR_STATE_INVALID, "calibration head is not fitted");
  const int T = n_tasks();
  for (int j = 0; j < n_blend; ++j)
    if (blend_task[j] < 0 || blend_task[j] >= T)
      fail(SR_ALIGNMENT, "blend references unknown task");  // service.cpp:258-262
  for (int b = 0; b + 1 < n_blocks; ++b)
    if (!(lo[b] <= hi[b] && hi[b] <= lo[b + 1]))
      fail(SR_PARAMETER, "calibration blocks must be sorted and disjoint");
  SR_CUDA_CHECK(cudaSetDevice(device_));
  std::vector<double> blk(static_cast<size_t>(3) * std::max(n_blocks, 1));
  for (int b = 0; b < n_blocks; ++b) {
    blk[3 * b] = lo[b];
    blk[3 * b + 1] = hi[b];
    blk[3 * b + 2] = value[b];
  }
  post_blocks_.ensure(blk.size());
  post_task_.ensure(static_cast<size_t>(std::max(n_blend, 1)));
  post_w_.ensure(static_cast<size_t>(std::max(n_blend, 1)));
  SR_CUDA_CHECK(cudaMemcpy(post_blocks_.ptr, blk.data(), blk.size() * sizeof(double),
                           cudaMemcpyHostToDevice));
  if (n_blend > 0) {
    SR_CUDA_CHECK(cudaMemcpy(post_task_.ptr, blend_task, n_blend * sizeof(int32_t),
                             cudaMemcpyHostToDevice));
    SR_CUDA_CHECK(cudaMemcpy(post_w_.ptr, blend_w, n_blend * sizeof(double),
                             cudaMemcpyHostToDevice));
  }
  post_nblocks_ = n_blocks;
  post_nblend_ = n_blend;
  post_on_ = n_blocks > 0 || n_blend > 0;
  last_final_.clear();
  ++ws_epoch_;  // captured graphs bake the launch list: re-capture
}

void Engine::ensure_workspace(int32_t M) {
  if (M <= ws_rows_) return;
  const int32_t rows = M + M / 4 + 128;
  const size_t d = cfg_.d_model, F = cfg_.d_ff;
  x_.release();
  xn_.release();
  qkv_.release();
  h_.release();
  xb_.release();
  stats_.release();
  ln_cnt_.release();
  // a failed allocation below leaves no workspace (not a stale size over freed
  // buffers), so the next call allocates again; captured graphs are stale
  ws_rows_ = 0;
  ++ws_epoch_;
  SR_CUDA_CHECK(cudaMalloc(&x_.ptr, rows * d * sizeof(float)));
  x_.cap = rows * d;
  SR_CUDA_CHECK(cudaMalloc(&xn_.ptr, rows * d * sizeof(__nv_bfloat16)));
  xn_.cap = rows * d;
  SR_CUDA_CHECK(cudaMalloc(&qkv_.ptr, rows * 3 * d * sizeof(__nv_bfloat16)));
  qkv_.cap = rows * 3 * d;
  SR_CUDA_CHECK(cudaMalloc(&h_.ptr, rows * F * sizeof(__nv_bfloat16)));
  h_.cap = rows * F;
  // Rows past M hold stale (always finite) data: GEMM tiles and attention key
  // blocks may read them, their results are masked or clipped, never stored.
  SR_CUDA_CHECK(cudaMemset(x_.ptr, 0, rows * d * sizeof(float)));
  SR_CUDA_CHECK(cudaMemset(qkv_.ptr, 0, rows * 3 * d * sizeof(__nv_bfloat16)));
  SR_CUDA_CHECK(cudaMemset(xn_.ptr, 0, rows * d * sizeof(__nv_bfloat16)));
  SR_CUDA_CHECK(cudaMemset(h_.ptr, 0, rows * F * sizeof(__nv_bfloat16)));
  SR_CUDA_CHECK(srk::make_tmap_bf16_2d(&tm_xn_, xn_.ptr, rows, d, 128, 64));
  SR_CUDA_CHECK(srk::make_tmap_bf16_2d(&tm_h_, h_.ptr, rows, F, 128, 64));
  SR_CUDA_CHECK(srk::make_tmap_bf16_2d(&tm_qkv_, qkv_.ptr, rows, 3 * d, 128, 64));
  if (fold_ln_) {
    SR_CUDA_CHECK(cudaMalloc(&xb_.ptr, rows * d * sizeof(__nv_bfloat16)));
    xb_.cap = rows * d;
    SR_CUDA_CHECK(cudaMemset(xb_.ptr, 0, rows * d * sizeof(__nv_bfloat16)));
    const size_t ns = (d / 128) * static_cast<size_t>(rows) * 2;
    SR_CUDA_CHECK(cudaMalloc(&stats_.ptr, ns * sizeof(float)));
    stats_.cap = ns;
    SR_CUDA_CHECK(cudaMemset(stats_.ptr, 0, ns * sizeof(float)));
    SR_CUDA_CHECK(srk::make_tmap_bf16_2d(&tm_xb_, xb_.ptr, rows, d, 128, 64));
  }
  if (ln_after_) {
    const size_t nb = static_cast<size_t>(rows) / 128 + 4;
    SR_CUDA_CHECK(cudaMalloc(&ln_cnt_.ptr, nb * sizeof(unsigned int)));
    ln_cnt_.cap = nb;
    SR_CUDA_CHECK(cudaMemset(ln_cnt_.ptr, 0, nb * sizeof(unsigned int)));
  }
  ws_rows_ = rows;
  ++ws_epoch_;
}

void Profiler::begin(int cls) {
  cudaEvent_t a;
  SR_CUDA_CHECK(cudaEventCreate(&a));
  // External record nodes: the events keep their timestamps inside a graph.
  SR_CUDA_CHECK(cudaEventRecordWithFlags(a, stream, in_graph ? cudaEventRecordExternal : 0));
  cur = cls;
  cur_start = a;
}
void Profiler::end() {
  cudaEvent_t b;
  SR_CUDA_CHECK(cudaEventCreate(&b));
  SR_CUDA_CHECK(cudaEventRecordWithFlags(b, stream, in_graph ? cudaEventRecordExternal : 0));
  marks.push_back({cur, {cur_start, b}});
}
Profiler::~Profiler() {
  for (auto& m : marks) {
    cudaEventDestroy(m.second.first);
    cudaEventDestroy(m.second.second);
  }
}

int32_t Engine::enqueue_forward(Plan& p, float* hidden_out, Profiler* prof) {
  const int M = p.pack.M, d = cfg_.d_model, F = cfg_.d_ff, H = cfg_.n_heads;
  const int hd = cfg_.head_dim();
  cudaStream_t s = stream_;
  int32_t n = 0;
  auto B = [&](int c) {
    if (prof) prof->begin(c);
  };
  auto E = [&]() {
    if (prof) prof->end();
  };
  auto attention = [&]() {
    if (hd >= 64)
      SR_CUDA_CHECK(srk::attention_tc(tm_qkv_, qkv_.ptr, p.spans.ptr, p.tiles.ptr,
                                      static_cast<int>(p.pack.tiles.size()), xn_.ptr, M, H, hd, s,
                                      p.n_attn_work ? p.attn_work.ptr : nullptr, p.n_attn_work));
    else  // toy head sizes (16/32): the 64-row mma.sync kernel
      SR_CUDA_CHECK(srk::attention(qkv_.ptr, p.spans.ptr, p.tiles.ptr,
                                   static_cast<int>(p.pack.tiles.size()), xn_.ptr, M, H, hd, s));
  };
  // Serpentine L2 order (SRK_SERPENTINE=0 disables): each kernel of the chain
  // O -> LN2 -> W_in -> W_out -> LN1 -> QKV walks its rows opposite to its
  // producer, so it starts on the rows still resident in L2.
  const bool serp = serpentine_;
  if (p.emb_form >= 0) {
    // compact embeddings -> soft rows in HBM, ahead of the embedding gather
    float* rows = p.soft.ptr + static_cast<size_t>(p.emb_row0) * d;
    B(PROF_EMBED_LN);
    if (p.emb_form == SR_EMB_PAD) {
      SR_CUDA_CHECK(srk::emb_pad_rows(p.emb.ptr, p.emb_n, p.emb_d, d, rows, s));
      ++n;
    } else {
      SR_CUDA_CHECK(srk::emb_to_bf16(p.emb.ptr, p.emb_n, p.emb_d, proj_kp_, p.emb16.ptr, s));
      const int N = proj_nsoft_ * d;
      SR_CUDA_CHECK(srk::gemm_auto(p.tm_emb16, tm_proj_, p.emb_n, N, proj_kp_, rows, N,
                                   srk::EPI_F32, s));
      n += 2;
    }
    E();
  }
  if (fold_ln_) {
    // LN folded into the GEMMs (gemm_tcgen05.cuh GemmLnArgs): no LayerNorm launches.
    srk::LnFold in{}, out{};
    in.stats_in = stats_.ptr;
    in.ld = ws_rows_;
    out.xb = xb_.ptr;
    out.stats_out = stats_.ptr;
    out.ld = ws_rows_;
    B(PROF_EMBED_LN);
    SR_CUDA_CHECK(srk::embed_stats(p.src.ptr, p.pos.ptr, tok_emb_,
                                   p.pack.n_soft ? p.soft.ptr : nullptr, pos_emb_, x_.ptr,
                                   xb_.ptr, stats_.ptr, M, d, s));
    E();
    ++n;
    for (int l = 0; l < cfg_.n_layers; ++l) {
      const auto& L = layers_[l];
      const bool last = l + 1 == cfg_.n_layers;
      in.n_parts = l == 0 ? 1 : d / 128;
      in.colsum = L.cs_qkv;
      B(PROF_GEMM_QKV);
      SR_CUDA_CHECK(srk::gemm_auto(tm_xb_, L.tm_qkv, M, 3 * d, d, qkv_.ptr, 3 * d,
                                   srk::EPI_LN_BF16, s, &in));
      E();
      B(PROF_ATTENTION);
      attention();
      E();
      B(PROF_GEMM_O);
      SR_CUDA_CHECK(srk::gemm_auto(tm_xn_, L.tm_o, M, d, d, x_.ptr, d, srk::EPI_RESID_LN, s, &out));
      E();
      in.n_parts = d / 128;
      in.colsum = L.cs_in;
      B(PROF_GEMM_IN);
      SR_CUDA_CHECK(srk::gemm_auto(tm_xb_, L.tm_in, M, F, d, h_.ptr, F, srk::EPI_LN_GELU_BF16, s,
                                   &in));
      E();
      // The last layer's x goes to the score head (final LN on fp32 rows):
      // no bf16 copy or statistics needed.
      B(PROF_GEMM_OUT);
      SR_CUDA_CHECK(srk::gemm_auto(tm_h_, L.tm_out, M, d, F, x_.ptr, d,
                                   last ? srk::EPI_RESID_F32 : srk::EPI_RESID_LN, s, &out));
      E();
      n += 5;
    }
  } else {
    // Residual GEMM (epilogue 7 counts finished 128-row blocks of x) with the
    // next LayerNorm in a concurrent kernel on the side stream that normalises
    // each block as soon as it is complete (x still in L2); joined before the
    // next projection reads xn.
    auto resid_ln = [&](const CUtensorMap& tm_a, const CUtensorMap& tm_w, int K, float* x,
                        const float* gain, int rows, bool rev) {
      srk::LnFold f{};
      f.ln_cnt = ln_cnt_.ptr;
      SR_CUDA_CHECK(cudaEventRecord(ev_fork_, s));
      SR_CUDA_CHECK(cudaStreamWaitEvent(side_, ev_fork_, 0));
      SR_CUDA_CHECK(srk::gemm_auto(tm_a, tm_w, rows, d, K, x, d, srk::EPI_RESID_F32_LN, s, &f, rev));
      SR_CUDA_CHECK(srk::layer_norm_after(x, gain, xn_.ptr, rows, d, ln_cnt_.ptr, d / 256, side_));
      SR_CUDA_CHECK(cudaEventRecord(ev_join_, side_));
      SR_CUDA_CHECK(cudaStreamWaitEvent(s, ev_join_, 0));
    };
    B(PROF_EMBED_LN);
    SR_CUDA_CHECK(srk::embed_ln(p.src.ptr, p.pos.ptr, tok_emb_, p.pack.n_soft ? p.soft.ptr : nullptr,
                                pos_emb_, layers_[0].ln1, x_.ptr, xn_.ptr, M, d, s));
    E();
    ++n;
    for (int l = 0; l < cfg_.n_layers; ++l) {
      const auto& L = layers_[l];
      B(PROF_GEMM_QKV);
      SR_CUDA_CHECK(srk::gemm_auto(tm_xn_, L.tm_qkv, M, 3 * d, d, qkv_.ptr, 3 * d, 0, s, nullptr,
                                   serp));
      E();
      B(PROF_ATTENTION);
      attention();
      E();
      B(PROF_GEMM_O);
      if (ln_after_) {  // x += attn . Wo, then LN2(x) -> xn by the last contributor
        resid_ln(tm_xn_, L.tm_o, d, x_.ptr, L.ln2, M, false);
        E();
        ++n;
      } else {
        SR_CUDA_CHECK(srk::gemm_auto(tm_xn_, L.tm_o, M, d, d, x_.ptr, d, 2, s));
        E();
        B(PROF_LAYERNORM);
        SR_CUDA_CHECK(srk::layer_norm_bf16(x_.ptr, L.ln2, xn_.ptr, M, d, s, serp));
        E();
        ++n;
      }
      B(PROF_GEMM_IN);
      SR_CUDA_CHECK(srk::gemm_auto(tm_xn_, L.tm_in, M, F, d, h_.ptr, F, 1, s));
      E();
      const bool next = l + 1 < cfg_.n_layers;
      B(PROF_GEMM_OUT);
      if (ln_after_ && next) {  // x += h . Wout, then LN1 of the next layer -> xn
        resid_ln(tm_h_, L.tm_out, F, x_.ptr, layers_[l + 1].ln1, M, serp);
        E();
        ++n;
      } else {
        SR_CUDA_CHECK(srk::gemm_auto(tm_h_, L.tm_out, M, d, F, x_.ptr, d, 2, s, nullptr, serp));
        E();
        if (next) {
          B(PROF_LAYERNORM);
          SR_CUDA_CHECK(srk::layer_norm_bf16(x_.ptr, layers_[l + 1].ln1, xn_.ptr, M, d, s));
          E();
          ++n;
        }
      }
      n += 5;
    }
  }
  B(PROF_SCORE_HEAD);
  SR_CUDA_CHECK(srk::score_head(x_.ptr, p.last_rows.ptr, p.pack.n_items, d, ln_f_, head_w_,
                                head_b_, n_cols_, task_col_, task_arity_, n_tasks(), yes_col_,
                                no_col_, p.scores.ptr, hidden_out, s));
  E();
  ++n;
  const double* key = p.scores.ptr;
  int key_stride = n_tasks();
  if (post_on_) {
    B(PROF_TOPK);
    SR_CUDA_CHECK(srk::final_scores(p.scores.ptr, n_tasks(), p.pack.n_items, post_blocks_.ptr,
                                    post_nblocks_, post_task_.ptr, post_w_.ptr, post_nblend_,
                                    p.final.ptr, s));
    E();
    ++n;
    key = p.final.ptr;
    key_stride = 1;
  }
  if (p.k > 0) {
    const int n_seg = static_cast<int>(p.pack.seg_off.size()) - 1;
    B(PROF_TOPK);
    SR_CUDA_CHECK(srk::topk(key, key_stride, p.ids.ptr, p.seg_off.ptr, n_seg,
                            p.pack.max_seg_len, p.k, p.topk_scratch.ptr,
                            static_cast<int>(p.topk_scratch.cap), p.topk_out.ptr, s));
    E();
    n += p.pack.max_seg_len > 4096 ? 2 : 1;
  }
  return n;
}

void Engine::profile(Plan& p, int reps, float* ms_out, int32_t* launches_out) {
  // Per-kernel-class device time as the plan's graph sees it: the forward is
  // captured once more with an event record node around every launch and
  // replayed (eager launches would add host launch gaps to every interval).
  SR_CUDA_CHECK(cudaSetDevice(device_));
  std::vector<double> acc(PROF_N, 0.0);
  std::vector<int32_t> cnt(PROF_N, 0);
  reps = std::max(reps, 1);
  Profiler prof;
  prof.stream = stream_;
  prof.in_graph = true;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  SR_CUDA_CHECK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue_forward(p, nullptr, &prof);
  } catch (...) {
    cudaStreamEndCapture(stream_, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  SR_CUDA_CHECK(cudaStreamEndCapture(stream_, &g));
  SR_CUDA_CHECK(cudaGraphInstantiate(&ge, g, 0));
  cudaGraphDestroy(g);
  SR_CUDA_CHECK(cudaGraphLaunch(ge, stream_));  // warm-up
  SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
  for (int r = 0; r < reps; ++r) {
    SR_CUDA_CHECK(cudaGraphLaunch(ge, stream_));
    SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
    for (auto& m : prof.marks) {
      float ms = 0.f;
      SR_CUDA_CHECK(cudaEventElapsedTime(&ms, m.second.first, m.second.second));
      acc[m.first] += ms;
      if (r == 0) cnt[m.first] += 1;
    }
  }
  cudaGraphExecDestroy(ge);
  for (int c = 0; c < PROF_N; ++c) {
    if (ms_out) ms_out[c] = static_cast<float>(acc[c] / reps);
    if (launches_out) launches_out[c] = cnt[c];
  }
}

namespace {
template <typename T, typename A>
void put(DevBuf<T>& b, const std::vector<T, A>& v, cudaStream_t s) {
  b.ensure(std::max<size_t>(v.size(), 1));
  if (!v.empty())
    SR_CUDA_CHECK(cudaMemcpyAsync(b.ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
}
}  // namespace

void Engine::refill_plan(Plan& p, const sr_request* reqs, int n_req) {
  SR_CUDA_CHECK(cudaSetDevice(device_));
  p.lens.resize(n_req);
  for (int q = 0; q < n_req; ++q) p.lens[q] = validate_request(cfg_, reqs[q]);
  p.reqs.assign(reqs, reqs + n_req);
  layout_signature(reqs, n_req, p.lens, sig_);
  const auto& pk = p.pack;
  if (layout_reuse_ && p.layout_ok && sig_ == p.layout_sig) {
    // same (t_q, mode, item lengths) as the arrays on the device: only the
    // token ids and doc ids change
    pack_sources(reqs, n_req, p.lens, p.pack);
    put(p.src, pk.row_src, stream_);
    put(p.ids, pk.ids, stream_);
  } else {
    p.layout_ok = false;
    pack_requests(cfg_, reqs, n_req, p.lens, p.pack);
    put(p.src, pk.row_src, stream_);
    put(p.pos, pk.row_pos, stream_);
    put(p.spans, pk.spans, stream_);
    put(p.tiles, pk.tiles, stream_);
    p.n_attn_work = 0;
    if (attn_lpt_ && cfg_.head_dim() >= 64 && !pk.tiles.empty()) {
      // longest-processing-time order of the (tile, head) items over the
      // persistent attention CTAs (attention_work_lpt)
      const int ctas = srk::attention_ctas(static_cast<int>(pk.tiles.size()), cfg_.n_heads, device_);
      srk::attention_work_lpt(pk.tiles.data(), static_cast<int>(pk.tiles.size()), cfg_.n_heads,
                              ctas, p.attn_work_host);
      put(p.attn_work, p.attn_work_host, stream_);
      p.n_attn_work = static_cast<int32_t>(p.attn_work_host.size());
    }
    put(p.last_rows, pk.last_rows, stream_);
    put(p.ids, pk.ids, stream_);
    put(p.seg_off, pk.seg_off, stream_);
    p.layout_sig.swap(sig_);
    p.layout_ok = true;
  }
  {
    // soft rows straight from the callers' buffers (one copy per request)
    const size_t d = cfg_.d_model;
    p.soft.ensure(std::max<size_t>(static_cast<size_t>(pk.n_soft) * d, 1));
    size_t off = 0;
    p.emb_form = -1;
    for (const auto& src : pk.soft_src) {
      if (src.rows == kEmbRows) {
        // compact embeddings: [n x d_emb] fp32 up, rows made in enqueue_forward
        const size_t ne = static_cast<size_t>(emb_.n) * emb_.d_emb;
        bool moved = p.emb.ensure(std::max<size_t>(ne, 1));
        up_.upload(p.emb.ptr, emb_.emb, ne * sizeof(float), stream_);
        if (emb_.form == SR_EMB_PROJECT) {
          const size_t rows = (static_cast<size_t>(emb_.n) + 127) / 128 * 128;
          if (p.emb16.ensure(rows * proj_kp_) || moved) {
            SR_CUDA_CHECK(srk::make_tmap_bf16_2d(&p.tm_emb16, p.emb16.ptr, rows, proj_kp_, 128, 64));
            moved = true;
          }
        }
        if (moved) p.graph_epoch = ~0ull;  // buffers baked into the graph moved
        p.emb_form = emb_.form;
        p.emb_n = emb_.n;
        p.emb_d = emb_.d_emb;
        p.emb_row0 = static_cast<int32_t>(off);
      } else if (src.rows == kB64Rows) {
        // base64 payloads: text to HBM, decoded in place into the rows
        const int32_t n = b64_.n;
        upload_b64_text();
        SR_CUDA_CHECK(srk::b64_decode(b64_text_.ptr, b64_off_.ptr, b64_off_.ptr + n,
                                      b64_off_.ptr + 2 * n, n,
                                      reinterpret_cast<uint8_t*>(p.soft.ptr + off * d),
                                      b64_err_.ptr, stream_));
      } else {
        up_.upload(p.soft.ptr + off * d, src.rows, src.n_rows * d * sizeof(float), stream_);
      }
      off += src.n_rows;
    }
  }
  p.scores.ensure(static_cast<size_t>(pk.n_items) * n_tasks());
  p.final.ensure(static_cast<size_t>(std::max(pk.n_items, 1)));
  const int n_seg = n_req;
  const int chunks = (pk.max_seg_len + 4095) / 4096;
  p.topk_scratch.ensure(static_cast<size_t>(std::max(1, n_seg * chunks * std::max(p.k, 1))));
  p.topk_out.ensure(static_cast<size_t>(std::max(1, n_seg * std::max(p.k, 1))));
  ensure_workspace(pk.M);
}

void Engine::capture(Plan& p) {
  if (p.graph) {
    cudaGraphExecDestroy(p.graph);
    p.graph = nullptr;
  }
  // Eager run first: sets kernel attributes outside capture and surfaces
  // launch errors with a precise location.
  p.launches = enqueue_forward(p, nullptr);
  SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
  cudaGraph_t g = nullptr;
  SR_CUDA_CHECK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue_forward(p, nullptr);
  } catch (...) {
    cudaStreamEndCapture(stream_, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  SR_CUDA_CHECK(cudaStreamEndCapture(stream_, &g));
  SR_CUDA_CHECK(cudaGraphInstantiate(&p.graph, g, 0));
  cudaGraphDestroy(g);
  p.graph_epoch = ws_epoch_;
}

std::unique_ptr<Plan> Engine::make_plan(const sr_request* reqs, int n_req, int32_t k) {
  if (k < 0) fail(SR_PARAMETER, "top-k must be >= 0");
  if (k > 4096) fail(SR_PARAMETER, "top-k must be <= 4096");
  auto p = std::make_unique<Plan>();
  p->eng = this;
  p->k = k;
  p->n_tasks = n_tasks();
  refill_plan(*p, reqs, n_req);
  const int chunks = (p->pack.max_seg_len + 4095) / 4096;
  if (k > 0 && chunks > 1 && static_cast<long>(chunks) * k > 4096)
    fail(SR_PARAMETER, "top-k too large for this many candidates");
  capture(*p);
  return p;
}

void Engine::run_plan(Plan& p) {
  SR_CUDA_CHECK(cudaSetDevice(device_));
  if (p.graph == nullptr || p.graph_epoch != ws_epoch_) capture(p);
  SR_CUDA_CHECK(cudaGraphLaunch(p.graph, stream_));
}

void Engine::fetch(Plan& p, sr_result* res, int n_req) {
  const auto& pk = p.pack;
  const int T = n_tasks();
  auto& scores = p.h_scores;
  auto& top = p.h_top;
  scores.resize(static_cast<size_t>(pk.n_items) * T);
  top.resize(static_cast<size_t>(n_req) * std::max(p.k, 0));
  SR_CUDA_CHECK(cudaMemcpyAsync(scores.data(), p.scores.ptr, scores.size() * sizeof(double),
                                cudaMemcpyDeviceToHost, stream_));
  if (post_on_) {
    last_final_.resize(static_cast<size_t>(pk.n_items));
    SR_CUDA_CHECK(cudaMemcpyAsync(last_final_.data(), p.final.ptr,
                                  last_final_.size() * sizeof(double), cudaMemcpyDeviceToHost,
                                  stream_));
  }
  if (p.k > 0)
    SR_CUDA_CHECK(cudaMemcpyAsync(top.data(), p.topk_out.ptr, top.size() * sizeof(srk::TopkEntry),
                                  cudaMemcpyDeviceToHost, stream_));
  SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
  for (int q = 0; q < n_req; ++q) {
    sr_result& r = res[q];
    const int32_t i0 = pk.seg_off[q], n = pk.seg_off[q + 1] - i0;
    if (r.scores)
      std::memcpy(r.scores, scores.data() + static_cast<size_t>(i0) * T,
                  static_cast<size_t>(n) * T * sizeof(double));
    const int32_t want = std::min(r.k, p.k);
    const int32_t kr = std::max(0, std::min(want, n));
    for (int32_t j = 0; j < kr; ++j) {
      const auto& e = top[static_cast<size_t>(q) * p.k + j];
      if (r.topk_ids) r.topk_ids[j] = e.id;
      if (r.topk_scores) r.topk_scores[j] = e.score;
      if (r.topk_index) r.topk_index[j] = e.index - i0;
    }
    r.k_returned = kr;
    report_for(cfg_, p.reqs[q], p.lens[q], &r.flops, &r.kv_incremental_per_item);
  }
}

void Engine::score(const sr_request* reqs, int n_req, sr_result* res) {
  if (n_req <= 0) fail(SR_SPEC_VIOLATION, "no requests");
  int32_t k = 0;
  for (int q = 0; q < n_req; ++q) k = std::max(k, res[q].k);
  // Shape key: packed rows, items, attention tiles, requests, longest
  // segment, soft rows, k. Same shape -> same captured graph.
  std::vector<std::vector<int32_t>> lens(n_req);
  int64_t M = 0, N = 0, soft = 0, tiles = 0;
  int32_t maxseg = 0;
  for (int q = 0; q < n_req; ++q) {
    lens[q] = validate_request(cfg_, reqs[q]);
    int64_t items = 0;
    for (int32_t l : lens[q]) items += l;
    M += reqs[q].t_q + items;
    N += reqs[q].n_items;
    const int tr = srk::attention_tile_rows(cfg_.head_dim());
    tiles += (reqs[q].t_q + tr - 1) / tr + (items + tr - 1) / tr;
    if (reqs[q].mode == SR_MODE_MIXED) soft += items;
    maxseg = std::max(maxseg, reqs[q].n_items);
  }
  const int32_t emb_key = emb_.form < 0 ? 0 : (emb_.form + 1) * 1000000 + emb_.d_emb;
  auto key = std::make_tuple(static_cast<int32_t>(M), static_cast<int32_t>(N),
                             static_cast<int32_t>(tiles), n_req, maxseg, static_cast<int32_t>(soft),
                             k, emb_key);
  auto it = cache_.find(key);
  Plan* p;
  if (it == cache_.end()) {
    if (cache_.size() >= 16) cache_.clear();
    auto np = make_plan(reqs, n_req, k);
    p = np.get();
    cache_[key] = std::move(np);
  } else {
    p = it->second.get();
    refill_plan(*p, reqs, n_req);
  }
  run_plan(*p);
  fetch(*p, res, n_req);
}

void Engine::upload_b64_text() {
  const int32_t n = b64_.n;
  const int64_t chars = b64_.la + b64_.lb;
  b64_text_.ensure(static_cast<size_t>(std::max<int64_t>(chars, 4)));
  b64_off_.ensure(static_cast<size_t>(3 * std::max(n, 1)));
  b64_err_.ensure(1);
  if (b64_.la > 0) up_.upload(b64_text_.ptr, b64_.a, static_cast<size_t>(b64_.la), stream_);
  if (b64_.lb > 0)
    up_.upload(b64_text_.ptr + b64_.la, b64_.b, static_cast<size_t>(b64_.lb), stream_);
  SR_CUDA_CHECK(cudaMemcpyAsync(b64_off_.ptr, b64_.spans.data(), b64_.spans.size() * sizeof(int64_t),
                                cudaMemcpyHostToDevice, stream_));
  SR_CUDA_CHECK(cudaMemsetAsync(b64_err_.ptr, 0xff, sizeof(unsigned long long), stream_));
}

void Engine::score_b64(const int32_t* prefix, int32_t t_q, const char* text,
                       const int64_t* char_off, int32_t n_items, const int64_t* item_ids,
                       sr_result* res) {
  std::vector<int64_t> begin(std::max(n_items, 0)), end(std::max(n_items, 0));
  for (int32_t j = 0; j < n_items; ++j) {
    begin[j] = char_off[j];
    end[j] = char_off[j + 1];
  }
  score_b64_spans(prefix, t_q, text, n_items > 0 ? char_off[n_items] : 0, nullptr, 0,
                  begin.data(), end.data(), n_items, item_ids, res);
}

void Engine::score_b64_spans(const int32_t* prefix, int32_t t_q, const char* a, int64_t la,
                             const char* b, int64_t lb, const int64_t* begin, const int64_t* end,
                             int32_t n_items, const int64_t* item_ids, sr_result* res) {
  if (n_items <= 0) fail(SR_PAYLOAD_INVALID, "request needs a non-empty items[]");
  const int64_t d = cfg_.d_model;
  auto at = [&](int64_t pos) { return pos < la ? a[pos] : b[pos - la]; };
  // Host-side checks in the reference's order per item (base64.cpp:60-64,
  // 97-101; service.cpp:365-369); character / padding checks run on the device.
  int bad = -1;
  std::string bad_msg;
  bool bad_before_chars = false;  // the length check precedes the character scan
  std::vector<int32_t> rows_off(n_items + 1, 0);
  std::vector<int64_t> byte_off(n_items + 1, 0);
  for (int32_t j = 0; j < n_items && bad < 0; ++j) {
    const int64_t len = end[j] - begin[j];
    if (len % 4 != 0) {
      bad = j;
      bad_msg = "base64 length must be mod 4";
      bad_before_chars = true;
      break;
    }
    const int pad = (len >= 1 && at(end[j] - 1) == '=') + (len >= 2 && at(end[j] - 2) == '=');
    const int64_t bytes = len / 4 * 3 - pad;
    if (bytes % 4 != 0) {
      bad = j;
      bad_msg = "payload is not a whole number of float32 values";
      break;
    }
    const int64_t floats = bytes / 4;
    if (floats == 0 || floats % d != 0) {
      bad = j;
      bad_msg = "embedding payload is not [n x " + std::to_string(d) + "] for item " +
                std::to_string(item_ids != nullptr ? item_ids[j] : j);
      break;
    }
    rows_off[j + 1] = rows_off[j] + static_cast<int32_t>(floats / d);
    byte_off[j + 1] = byte_off[j] + bytes;
  }
  SR_CUDA_CHECK(cudaSetDevice(device_));
  b64_.a = a;
  b64_.la = la;
  b64_.b = b;
  b64_.lb = lb;
  b64_.n = n_items;
  b64_.spans.assign(begin, begin + n_items);
  b64_.spans.insert(b64_.spans.end(), end, end + n_items);
  b64_.spans.insert(b64_.spans.end(), byte_off.begin(), byte_off.begin() + n_items);
  auto raise_char = [](unsigned long long err) {
    fail(SR_PAYLOAD_INVALID, (err & 3u) == 1u ? "misplaced base64 padding"
                                              : "invalid base64 character");
  };
  if (bad >= 0) {
    // validate-only pass over the items the reference would have decoded
    const int32_t upto = bad_before_chars ? bad : bad + 1;
    unsigned long long err = ~0ull;
    if (upto > 0) {
      upload_b64_text();
      SR_CUDA_CHECK(srk::b64_decode(b64_text_.ptr, b64_off_.ptr, b64_off_.ptr + n_items,
                                    b64_off_.ptr + 2 * n_items, upto, nullptr, b64_err_.ptr,
                                    stream_));
      SR_CUDA_CHECK(cudaMemcpyAsync(&err, b64_err_.ptr, sizeof(err), cudaMemcpyDeviceToHost,
                                    stream_));
      SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
    }
    b64_ = B64Src{};
    if (err != ~0ull) raise_char(err);
    fail(SR_PAYLOAD_INVALID, bad_msg);
  }
  // item_offsets index soft rows; the rows come from the base64 text
  sr_request req{};
  req.prefix_tokens = prefix;
  req.t_q = t_q;
  req.n_items = n_items;
  req.item_offsets = rows_off.data();
  req.item_tokens = nullptr;
  req.item_rows = kB64Rows;
  req.item_ids = item_ids;
  req.mode = SR_MODE_MIXED;
  try {
    score(&req, 1, res);
  } catch (...) {
    b64_ = B64Src{};
    throw;
  }
  b64_ = B64Src{};
  unsigned long long err = ~0ull;
  SR_CUDA_CHECK(cudaMemcpy(&err, b64_err_.ptr, sizeof(err), cudaMemcpyDeviceToHost));
  if (err != ~0ull) raise_char(err);  // results are discarded, as the reference never scores
}

void Engine::set_projection(const float* proj, int32_t d_emb, int32_t n_soft) {
  SR_CUDA_CHECK(cudaSetDevice(device_));
  SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
  if (proj == nullptr) {  // remove
    proj_.release();
    proj_demb_ = proj_kp_ = proj_nsoft_ = 0;
    ++ws_epoch_;
    return;
  }
  const int d = cfg_.d_model;
  if (d_emb < 1 || n_soft < 1) fail(SR_PARAMETER, "projection needs d_emb >= 1 and n_soft >= 1");
  if (n_soft > cfg_.max_seq) fail(SR_LENGTH_OVERFLOW, "n_soft exceeds max_seq");
  const int kp = (d_emb + 63) / 64 * 64;
  const size_t N = static_cast<size_t>(n_soft) * d;
  // reference layout [d_emb x N] (weights are [d_in x d_out], model.hpp:42-47)
  // -> zero-padded [kp x N] -> bf16 [N x kp] (K-major B operand)
  std::vector<float> padded(static_cast<size_t>(kp) * N, 0.f);
  std::memcpy(padded.data(), proj, static_cast<size_t>(d_emb) * N * sizeof(float));
  float* stage = nullptr;
  SR_CUDA_CHECK(cudaMalloc(&stage, padded.size() * sizeof(float)));
  try {
    proj_.ensure(padded.size());
    SR_CUDA_CHECK(cudaMemcpyAsync(stage, padded.data(), padded.size() * sizeof(float),
                                  cudaMemcpyHostToDevice, stream_));
    SR_CUDA_CHECK(srk::transpose_to_bf16(stage, proj_.ptr, kp, static_cast<int>(N), stream_,
                                         nullptr));
    SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
  } catch (...) {
    cudaFree(stage);
    throw;
  }
  cudaFree(stage);
  make_weight_map(&tm_proj_, proj_.ptr, static_cast<int>(N), kp);
  proj_demb_ = d_emb;
  proj_kp_ = kp;
  proj_nsoft_ = n_soft;
  ++ws_epoch_;  // captured projection graphs bake the old operand
}

std::vector<int32_t> Engine::emb_request(const int32_t* prefix, int32_t t_q, const float* emb,
                                         int32_t d_emb, int32_t n_items, const int64_t* item_ids,
                                         int32_t form, sr_request* req) {
  if (form != SR_EMB_PAD && form != SR_EMB_PROJECT)
    fail(SR_PARAMETER, "unknown embedding form " + std::to_string(form));
  if (n_items <= 0) fail(SR_PAYLOAD_INVALID, "request needs a non-empty items[]");
  if (emb == nullptr) fail(SR_SPEC_VIOLATION, "null embeddings");
  int32_t rows = 1;
  if (form == SR_EMB_PAD) {
    if (d_emb < 1) fail(SR_PAYLOAD_INVALID, "embedding must have at least one value");
  } else {
    if (proj_nsoft_ == 0) fail(SR_STATE_INVALID, "no embedding projection is set");
    if (d_emb != proj_demb_)
      fail(SR_ALIGNMENT, "embedding width " + std::to_string(d_emb) +
                             " differs from the projection's " + std::to_string(proj_demb_));
    rows = proj_nsoft_;
  }
  std::vector<int32_t> off(static_cast<size_t>(n_items) + 1);
  for (int32_t j = 0; j <= n_items; ++j) off[j] = j * rows;
  *req = sr_request{};
  req->prefix_tokens = prefix;
  req->t_q = t_q;
  req->n_items = n_items;
  req->item_offsets = off.data();
  req->item_rows = kEmbRows;
  req->item_ids = item_ids;
  req->mode = SR_MODE_MIXED;
  emb_ = EmbSrc{emb, n_items, d_emb, form};
  return off;
}

void Engine::score_emb(const int32_t* prefix, int32_t t_q, const float* emb, int32_t d_emb,
                       int32_t n_items, const int64_t* item_ids, int32_t form, sr_result* res) {
  sr_request req;
  const auto off = emb_request(prefix, t_q, emb, d_emb, n_items, item_ids, form, &req);
  try {
    score(&req, 1, res);
  } catch (...) {
    emb_ = EmbSrc{};
    throw;
  }
  emb_ = EmbSrc{};
}

std::unique_ptr<Plan> Engine::make_plan_emb(const int32_t* prefix, int32_t t_q, const float* emb,
                                            int32_t d_emb, int32_t n_items,
                                            const int64_t* item_ids, int32_t form, int32_t k) {
  sr_request req;
  const auto off = emb_request(prefix, t_q, emb, d_emb, n_items, item_ids, form, &req);
  std::unique_ptr<Plan> p;
  try {
    p = make_plan(&req, 1, k);
  } catch (...) {
    emb_ = EmbSrc{};
    throw;
  }
  emb_ = EmbSrc{};
  // the plan keeps the request; its offsets must outlive this call
  p->emb_off = off;
  p->reqs[0].item_offsets = p->emb_off.data();
  return p;
}

void Engine::item_hidden(const sr_request& req, float* hidden_out) {
  auto p = std::make_unique<Plan>();
  p->eng = this;
  p->k = 0;
  refill_plan(*p, &req, 1);
  float* dh = nullptr;
  const size_t n = static_cast<size_t>(p->pack.n_items) * cfg_.d_model;
  SR_CUDA_CHECK(cudaMalloc(&dh, n * sizeof(float)));
  try {
    enqueue_forward(*p, dh);
    SR_CUDA_CHECK(cudaMemcpyAsync(hidden_out, dh, n * sizeof(float), cudaMemcpyDeviceToHost, stream_));
    SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
  } catch (...) {
    cudaFree(dh);
    throw;
  }
  cudaFree(dh);
}

void Engine::run_plan_sharded(Plan& p, Comm* c) {
  // nranks == 1 also takes the all-gather + merge (a copy): one code path,
  // exercised by the single-GPU tests
  if (c == nullptr) {
    run_plan(p);
    return;
  }
  if (p.k <= 0) fail(SR_PARAMETER, "sharded scoring needs k >= 1");
  if (p.reqs.size() != 1) fail(SR_PARAMETER, "sharded scoring takes one request per call");
  if (static_cast<long>(c->nranks) * p.k > 4096) fail(SR_PARAMETER, "nranks * k must be <= 4096");
  run_plan(p);
  p.gathered.ensure(static_cast<size_t>(c->nranks) * p.k);
  p.merged.ensure(static_cast<size_t>(p.k));
  nccl_allgather_bytes(c, p.topk_out.ptr, p.gathered.ptr, sizeof(srk::TopkEntry) * p.k, stream_);
  SR_CUDA_CHECK(srk::topk_merge(p.gathered.ptr, c->nranks * p.k, p.k, p.merged.ptr, stream_));
}

// ------------------------------------------------------------------- NCCL
namespace {
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // Prefer an already-loaded libnccl (e.g. torch's), else the system one.
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.lib = h;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank =
        reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.error_string =
        reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.lib || !api.get_unique_id || !api.comm_init_rank || !api.all_gather)
    fail(SR_NCCL, "libnccl.so.2 not loadable");
  return api;
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(SR_NCCL, std::string(what) + ": " +
                      (nccl().error_string ? nccl().error_string(r) : "nccl error"));
}
}  // namespace

void nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

Comm* comm_create(int nranks, int rank, const uint8_t id[128], int device) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(SR_PARAMETER, "bad rank/nranks");
  SR_CUDA_CHECK(cudaSetDevice(device));
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, 128);
  auto* c = new Comm;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ncclComm_t comm = nullptr;
  try {
    nccl_check(nccl().comm_init_rank(&comm, nranks, uid, rank), "ncclCommInitRank");
  } catch (...) {
    delete c;
    throw;
  }
  c->nccl = comm;
  return c;
}

Comm* comm_create_host(int nranks, int rank, int device, sr_allgather_fn fn, void* user) {
  if (nranks < 1 || rank < 0 || rank >= nranks) fail(SR_PARAMETER, "bad rank/nranks");
  if (fn == nullptr) fail(SR_SPEC_VIOLATION, "null all-gather callback");
  auto* c = new Comm;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  c->host_fn = fn;
  c->host_user = user;
  return c;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->nccl && nccl().comm_destroy) nccl().comm_destroy(static_cast<ncclComm_t>(c->nccl));
  delete c;
}

void nccl_allgather_bytes(Comm* c, const void* send, void* recv, size_t bytes, cudaStream_t s) {
  if (c->host_fn != nullptr) {
    // the caller's transport: this rank's bytes out, every rank's bytes back
    std::vector<uint8_t> hs(bytes), hr(bytes * static_cast<size_t>(c->nranks));
    SR_CUDA_CHECK(cudaMemcpyAsync(hs.data(), send, bytes, cudaMemcpyDeviceToHost, s));
    SR_CUDA_CHECK(cudaStreamSynchronize(s));
    if (c->host_fn(hs.data(), hr.data(), bytes, c->host_user) != 0)
      fail(SR_NCCL, "host all-gather callback failed");
    SR_CUDA_CHECK(cudaMemcpyAsync(recv, hr.data(), hr.size(), cudaMemcpyHostToDevice, s));
    SR_CUDA_CHECK(cudaStreamSynchronize(s));
    return;
  }
  nccl_check(nccl().all_gather(send, recv, bytes, ncclUint8, static_cast<ncclComm_t>(c->nccl), s),
             "ncclAllGather");
}

void Engine::rank(const double* h_scores, const int64_t* ids, int32_t n, sr_result* res) {
  SR_CUDA_CHECK(cudaSetDevice(device_));
  const int T = n_tasks();
  if (res->k < 0) fail(SR_PARAMETER, "top-k must be >= 0");
  const int32_t k = std::min(res->k, n);
  if (res->scores && res->scores != h_scores)
    std::memcpy(res->scores, h_scores, static_cast<size_t>(n) * T * sizeof(double));
  res->k_returned = k;
  last_final_.clear();
  if (n == 0 || (k == 0 && !post_on_)) return;
  if (k > 4096) fail(SR_PARAMETER, "top-k must be <= 4096");
  const int chunks = (n + 4095) / 4096;
  if (k > 0 && chunks > 1 && static_cast<long>(chunks) * k > 4096)
    fail(SR_PARAMETER, "top-k too large for this many candidates");
  rk_scores_.ensure(static_cast<size_t>(n) * T);
  rk_final_.ensure(static_cast<size_t>(n));
  rk_ids_.ensure(static_cast<size_t>(n));
  rk_seg_.ensure(2);
  rk_scratch_.ensure(static_cast<size_t>(chunks) * std::max(k, 1));
  rk_out_.ensure(static_cast<size_t>(std::max(k, 1)));
  const int32_t seg[2] = {0, n};
  SR_CUDA_CHECK(cudaMemcpyAsync(rk_scores_.ptr, h_scores, static_cast<size_t>(n) * T * sizeof(double),
                                cudaMemcpyHostToDevice, stream_));
  SR_CUDA_CHECK(cudaMemcpyAsync(rk_ids_.ptr, ids, static_cast<size_t>(n) * sizeof(int64_t),
                                cudaMemcpyHostToDevice, stream_));
  SR_CUDA_CHECK(cudaMemcpyAsync(rk_seg_.ptr, seg, sizeof(seg), cudaMemcpyHostToDevice, stream_));
  const double* key = rk_scores_.ptr;
  int stride = T;
  if (post_on_) {
    SR_CUDA_CHECK(srk::final_scores(rk_scores_.ptr, T, n, post_blocks_.ptr, post_nblocks_,
                                    post_task_.ptr, post_w_.ptr, post_nblend_, rk_final_.ptr,
                                    stream_));
    key = rk_final_.ptr;
    stride = 1;
  }
  std::vector<srk::TopkEntry> top(static_cast<size_t>(k));
  if (k > 0) {
    SR_CUDA_CHECK(srk::topk(key, stride, rk_ids_.ptr, rk_seg_.ptr, 1, n, k, rk_scratch_.ptr,
                            static_cast<int>(rk_scratch_.cap), rk_out_.ptr, stream_));
    SR_CUDA_CHECK(cudaMemcpyAsync(top.data(), rk_out_.ptr, top.size() * sizeof(srk::TopkEntry),
                                  cudaMemcpyDeviceToHost, stream_));
  }
  if (post_on_) {
    last_final_.resize(static_cast<size_t>(n));
    SR_CUDA_CHECK(cudaMemcpyAsync(last_final_.data(), rk_final_.ptr, n * sizeof(double),
                                  cudaMemcpyDeviceToHost, stream_));
  }
  SR_CUDA_CHECK(cudaStreamSynchronize(stream_));
  for (int32_t j = 0; j < k; ++j) {
    if (res->topk_ids) res->topk_ids[j] = top[j].id;
    if (res->topk_scores) res->topk_scores[j] = top[j].score;
    if (res->topk_index) res->topk_index[j] = top[j].index;
  }
}

void Engine::score_cached(ScoreCache& cache, const std::string& searcher_id, uint64_t signature,
                          const std::string& model_version, const sr_request& req,
                          sr_result* res, int32_t* n_hits) {
  if (req.item_ids == nullptr)
    fail(SR_SPEC_VIOLATION, "cached scoring needs item_ids (the cache keys' entity ids)");
  if (req.n_items < 1) fail(SR_SPEC_VIOLATION, "request has no items");
  if (req.item_offsets == nullptr) fail(SR_SPEC_VIOLATION, "item_offsets is null");
  if (res->k < 0) fail(SR_PARAMETER, "top-k must be >= 0");
  if (res->k > 4096) fail(SR_PARAMETER, "top-k must be <= 4096");
  const int T = n_tasks();
  const int32_t n = req.n_items;
  std::vector<double> rows(static_cast<size_t>(n) * T);
  std::vector<int32_t> miss;
  CacheKey key{searcher_id, signature, 0, model_version};
  for (int32_t i = 0; i < n; ++i) {  // probe everything first (service.cpp:166-180)
    key.entity_id = req.item_ids[i];
    if (!cache.get(key, rows.data() + static_cast<size_t>(i) * T, T)) miss.push_back(i);
  }
  if (n_hits) *n_hits = n - static_cast<int32_t>(miss.size());
  if (!miss.empty()) {
    // The misses as one request, in request order (service.cpp:196-221).
    const bool mixed = req.mode == SR_MODE_MIXED;
    const int64_t width = mixed ? cfg_.d_model : 1;
    const int32_t m = static_cast<int32_t>(miss.size());
    std::vector<int32_t> off(static_cast<size_t>(m) + 1, 0);
    std::vector<int64_t> ids(static_cast<size_t>(m));
    for (int32_t j = 0; j < m; ++j) {
      const int32_t i = miss[j];
      const int32_t len = req.item_offsets[i + 1] - req.item_offsets[i];
      if (len < 0) fail(SR_SPEC_VIOLATION, "item_offsets must be non-decreasing");
      off[j + 1] = off[j] + len;
      ids[j] = req.item_ids[i];
    }
    std::vector<int32_t> toks;
    std::vector<float> soft;
    sr_request sub = req;
    sub.n_items = m;
    sub.item_offsets = off.data();
    sub.item_ids = ids.data();
    if (m == n) {
      sub.item_tokens = req.item_tokens;
      sub.item_rows = req.item_rows;
    } else if (mixed) {
      if (req.item_rows == nullptr) fail(SR_SPEC_VIOLATION, "item_rows is null");
      soft.resize(static_cast<size_t>(off[m]) * width);
      for (int32_t j = 0; j < m; ++j)
        std::memcpy(soft.data() + static_cast<size_t>(off[j]) * width,
                    req.item_rows + static_cast<size_t>(req.item_offsets[miss[j]]) * width,
                    static_cast<size_t>(off[j + 1] - off[j]) * width * sizeof(float));
      sub.item_rows = soft.data();
    } else {
      if (req.item_tokens == nullptr) fail(SR_SPEC_VIOLATION, "item_tokens is null");
      toks.resize(static_cast<size_t>(off[m]));
      for (int32_t j = 0; j < m; ++j)
        std::memcpy(toks.data() + off[j], req.item_tokens + req.item_offsets[miss[j]],
                    static_cast<size_t>(off[j + 1] - off[j]) * sizeof(int32_t));
      sub.item_tokens = toks.data();
    }
    std::vector<double> got(static_cast<size_t>(m) * T);
    sr_result sr{};
    sr.scores = got.data();
    score(&sub, 1, &sr);
    res->flops = sr.flops;
    res->kv_incremental_per_item = sr.kv_incremental_per_item;
    for (int32_t j = 0; j < m; ++j) {  // service.cpp:225-233
      std::memcpy(rows.data() + static_cast<size_t>(miss[j]) * T, got.data() + static_cast<size_t>(j) * T,
                  T * sizeof(double));
      key.entity_id = ids[j];
      cache.put(key, got.data() + static_cast<size_t>(j) * T, T);
    }
  } else {
    res->flops = sr_flop_report{};
    res->kv_incremental_per_item = 0.0;
  }
  rank(rows.data(), req.item_ids, n, res);
}

}  // namespace srh
