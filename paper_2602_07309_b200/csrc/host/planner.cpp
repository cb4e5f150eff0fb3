#include "planner.hpp"

#include <algorithm>
#include <numeric>
#include <string>

namespace srh {

namespace {

sr_flop_report actual_flops(bool amortized, double tq, const std::vector<int32_t>& lens) {
  // engine.cpp:63-88
  sr_flop_report r{};
  r.t_q = tq;
  r.n_items = static_cast<double>(lens.size());
  double sum = 0;
  for (int32_t l : lens) sum += l;
  r.t_i_mean = lens.empty() ? 0 : sum / r.n_items;
  if (amortized) {
    r.attention_units = tq * tq;
    r.linear_units = tq;
    for (int32_t l : lens) {
      const double ti = l;
      r.attention_units += 2.0 * ti * tq + ti * ti;
      r.linear_units += ti;
    }
  } else {
    for (int32_t l : lens) {
      const double ti = l;
      r.attention_units += (tq + ti) * (tq + ti);
      r.linear_units += tq + ti;
    }
  }
  return r;
}
}  // namespace

sr_flop_report flops(int mode, int64_t t_q, int64_t t_i, int64_t n_items) {  // engine.cpp:30-47
  if (t_q < 0 || t_i < 0 || n_items < 0) fail(SR_PARAMETER, "flop counts must be non-negative");
  if (mode < SR_MODE_NAIVE || mode > SR_MODE_MIXED) fail(SR_PARAMETER, "unknown scoring mode");
  sr_flop_report r{};
  r.t_q = static_cast<double>(t_q);
  r.t_i_mean = static_cast<double>(t_i);
  r.n_items = static_cast<double>(n_items);
  const double tq = r.t_q, ti = r.t_i_mean, n = r.n_items;
  if (mode == SR_MODE_NAIVE) {
    r.attention_units = n * (tq + ti) * (tq + ti);
    r.linear_units = n * (tq + ti);
  } else {
    r.attention_units = tq * tq + n * (2.0 * ti * tq + ti * ti);
    r.linear_units = tq + n * ti;
  }
  return r;
}

std::vector<int32_t> validate_request(const ModelConfig& cfg, const sr_request& req) {
  if (req.mode < SR_MODE_NAIVE || req.mode > SR_MODE_MIXED)
    fail(SR_PARAMETER, "unknown scoring mode");  // engine.cpp:28
  if (req.n_items <= 0) fail(SR_SPEC_VIOLATION, "request has no items");
  if (req.t_q < 0) fail(SR_SPEC_VIOLATION, "negative prefix length");
  if (req.t_q > 0 && req.prefix_tokens == nullptr)
    fail(SR_SPEC_VIOLATION, "prefix_tokens is null");
  if (req.item_offsets == nullptr) fail(SR_SPEC_VIOLATION, "item_offsets is null");
  if (req.item_offsets[0] != 0) fail(SR_SPEC_VIOLATION, "item_offsets[0] must be 0");
  const bool mixed = req.mode == SR_MODE_MIXED;
  std::vector<int32_t> lens(req.n_items);
  for (int i = 0; i < req.n_items; ++i) {
    const int32_t len = req.item_offsets[i + 1] - req.item_offsets[i];
    if (mixed) {
      // engine.cpp:243-251: n_emb_tokens >= 1 and payload [n x d]
      if (len < 1)
        fail(SR_PAYLOAD_INVALID, "item " + std::to_string(i) + " embedding payload is not [n x " +
                                     std::to_string(cfg.d_model) + "]");
    } else if (len < 1) {
      // engine.cpp:51-61 require_token_mode
      fail(SR_SPEC_VIOLATION, "token-mode item has no tokens: " + std::to_string(i));
    }
    lens[i] = len;
  }
  if (mixed && req.item_rows == nullptr) fail(SR_PAYLOAD_INVALID, "mixed request without rows");
  if (!mixed && req.item_tokens == nullptr) fail(SR_SPEC_VIOLATION, "item_tokens is null");
  // Token range (model.cpp:260-264) for prefix and items.
  auto check_tok = [&](int32_t t) {
    if (t < 0 || t >= cfg.vocab_size)
      fail(SR_SPEC_VIOLATION, "token id " + std::to_string(t) + " out of vocabulary");
  };
  // Capacity (model.cpp:222-247): the prefix alone, then prefix + each item,
  // must fit max_seq — every mode prefills T_q then T_i rows per item
  // (chunked multi-item: engine.cpp:340-343 "cannot fit max_seq even alone").
  if (req.t_q > cfg.max_seq)
    fail(SR_LENGTH_OVERFLOW, "prefill of " + std::to_string(req.t_q) +
                                 " tokens after 0 would exceed max_seq " +
                                 std::to_string(cfg.max_seq));
  for (int j = 0; j < req.t_q; ++j) check_tok(req.prefix_tokens[j]);
  for (int i = 0; i < req.n_items; ++i) {
    if (static_cast<int64_t>(req.t_q) + lens[i] > cfg.max_seq)
      fail(SR_LENGTH_OVERFLOW, "item " + std::to_string(i) + " cannot fit max_seq even alone");
    if (!mixed)
      for (int32_t j = req.item_offsets[i]; j < req.item_offsets[i + 1]; ++j)
        check_tok(req.item_tokens[j]);
  }
  return lens;
}

void report_for(const ModelConfig& cfg, const sr_request& req, const std::vector<int32_t>& lens,
                sr_flop_report* flops_out, double* kv_out) {
  const double tq = req.t_q;
  const double n = static_cast<double>(lens.size());
  double ti_sum = 0;
  for (int32_t l : lens) ti_sum += l;
  sr_flop_report r{};
  double kv = 0;
  switch (req.mode) {
    case SR_MODE_NAIVE:  // engine.cpp:100-121
      r = actual_flops(false, tq, lens);
      kv = (n * tq + ti_sum) / n;
      break;
    case SR_MODE_IBPC:   // engine.cpp:123-145
    case SR_MODE_MIXED:  // engine.cpp:238-276
      r = actual_flops(true, tq, lens);
      kv = ti_sum / n;
      break;
    case SR_MODE_MULTI_ITEM: {  // engine.cpp:328-377 (chunked; each chunk repays the prefix)
      std::vector<std::pair<size_t, size_t>> chunks;
      size_t begin = 0;
      int64_t used = req.t_q;
      for (size_t i = 0; i < lens.size(); ++i) {
        if (used + lens[i] > cfg.max_seq) {
          chunks.emplace_back(begin, i);
          begin = i;
          used = req.t_q;
        }
        used += lens[i];
      }
      chunks.emplace_back(begin, lens.size());
      if (chunks.size() == 1) {
        r = actual_flops(true, tq, lens);
      } else {
        for (const auto& [lo, hi] : chunks) {
          std::vector<int32_t> part(lens.begin() + lo, lens.begin() + hi);
          const auto c = actual_flops(true, tq, part);
          r.attention_units += c.attention_units;
          r.linear_units += c.linear_units;
        }
        r.t_q = tq;
        r.n_items = n;
        r.t_i_mean = ti_sum / n;
      }
      kv = ti_sum / n;
      break;
    }
  }
  if (flops_out) *flops_out = r;
  if (kv_out) *kv_out = kv;
}

void pack_requests(const ModelConfig& cfg, const sr_request* reqs, int n_req,
                   const std::vector<std::vector<int32_t>>& lens, PackedBatch& out) {
  const int d = cfg.d_model;
  const int kTileRows = srk::attention_tile_rows(cfg.head_dim());
  int64_t M = 0, N = 0, R = 0;
  for (int q = 0; q < n_req; ++q) {
    M += reqs[q].t_q;
    for (int32_t l : lens[q]) M += l;
    N += reqs[q].n_items;
    if (reqs[q].mode == SR_MODE_MIXED) R += reqs[q].item_offsets[reqs[q].n_items];
  }
  if (M > INT32_MAX / 4) fail(SR_LENGTH_OVERFLOW, "packed batch too large");
  out.M = static_cast<int32_t>(M);
  out.n_items = static_cast<int32_t>(N);
  out.row_src.resize(M);
  out.row_pos.resize(M);
  out.spans.resize(M);
  out.tiles.clear();
  out.last_rows.resize(N);
  out.ids.resize(N);
  out.seg_off.assign(n_req + 1, 0);
  out.soft_src.clear();
  out.n_soft = static_cast<int32_t>(R);
  out.max_seg_len = 0;

  int32_t row = 0, item = 0, soft = 0;
  for (int q = 0; q < n_req; ++q) {
    const sr_request& rq = reqs[q];
    const int32_t base = row;
    const int32_t tq = rq.t_q;
    for (int32_t j = 0; j < tq; ++j, ++row) {
      out.row_src[row] = rq.prefix_tokens[j];
      out.row_pos[row] = j;
      out.spans[row] = {base, base, base, 0};
    }
    for (int32_t r0 = base; r0 < base + tq; r0 += kTileRows) {
      const int32_t r1 = std::min(r0 + kTileRows, base + tq);
      out.tiles.push_back({r0, r1, 0, 0, base, r1, 0, 0});
    }
    const int32_t items_begin = row;
    const bool mixed = rq.mode == SR_MODE_MIXED;
    if (mixed && rq.n_items > 0)
      out.soft_src.push_back({rq.item_rows, static_cast<size_t>(rq.item_offsets[rq.n_items])});
    for (int i = 0; i < rq.n_items; ++i) {
      const int32_t s = row, L = lens[q][i];
      for (int32_t j = 0; j < L; ++j, ++row) {
        if (mixed) {
          // soft row index == this request's row index rq.item_offsets[i] + j,
          // offset by the rows of earlier requests
          out.row_src[row] = -(1 + soft);
          ++soft;
        } else {
          out.row_src[row] = rq.item_tokens[rq.item_offsets[i] + j];
        }
        out.row_pos[row] = tq + j;  // prefix-relative positions (engine.cpp:209-217)
        out.spans[row] = {base, base + tq, s, 0};
      }
      out.last_rows[item] = s + L - 1;
      out.ids[item] = rq.item_ids != nullptr ? rq.item_ids[i] : static_cast<int64_t>(i);
      ++item;
    }
    for (int32_t r0 = items_begin; r0 < row; r0 += kTileRows) {
      const int32_t r1 = std::min(r0 + kTileRows, row);
      out.tiles.push_back({r0, r1, base, base + tq, out.spans[r0].span_start, r1, 0, 0});
    }
    out.seg_off[q + 1] = item;
    out.max_seg_len = std::max(out.max_seg_len, rq.n_items);
  }
}

void layout_signature(const sr_request* reqs, int n_req,
                      const std::vector<std::vector<int32_t>>& lens, std::vector<int32_t>& sig) {
  sig.clear();
  sig.push_back(n_req);
  for (int q = 0; q < n_req; ++q) {
    sig.push_back(reqs[q].t_q);
    sig.push_back(reqs[q].mode == SR_MODE_MIXED);
    sig.push_back(reqs[q].n_items);
    sig.insert(sig.end(), lens[q].begin(), lens[q].end());
  }
}

void pack_sources(const sr_request* reqs, int n_req,
                  const std::vector<std::vector<int32_t>>& lens, PackedBatch& out) {
  out.soft_src.clear();
  int32_t row = 0, item = 0;
  for (int q = 0; q < n_req; ++q) {
    const sr_request& rq = reqs[q];
    std::copy(rq.prefix_tokens, rq.prefix_tokens + rq.t_q, out.row_src.begin() + row);
    row += rq.t_q;
    const bool mixed = rq.mode == SR_MODE_MIXED;
    if (mixed && rq.n_items > 0)
      out.soft_src.push_back({rq.item_rows, static_cast<size_t>(rq.item_offsets[rq.n_items])});
    for (int i = 0; i < rq.n_items; ++i) {
      const int32_t L = lens[q][i];
      if (!mixed)  // mixed rows keep their soft-row indices (layout only)
        std::copy(rq.item_tokens + rq.item_offsets[i], rq.item_tokens + rq.item_offsets[i] + L,
                  out.row_src.begin() + row);
      row += L;
      out.ids[item++] = rq.item_ids != nullptr ? rq.item_ids[i] : static_cast<int64_t>(i);
    }
  }
}

int64_t multi_item_pair_count(int32_t prefix_len, const int32_t* lens, int n) {
  // engine.cpp:147-155
  const int64_t tq = prefix_len;
  int64_t count = tq * (tq + 1) / 2;
  for (int i = 0; i < n; ++i) {
    const int64_t len = lens[i];
    count += tq * len + len * (len + 1) / 2;
  }
  return count;
}

std::vector<Batch> plan_batches(const std::vector<int32_t>& prefix_len,
                                const std::vector<std::vector<int32_t>>& item_len,
                                int64_t max_batch_tokens) {  // engine.cpp:278-326
  std::vector<Batch> batches;
  Batch cur;
  auto flush = [&] {
    if (!cur.entries.empty()) {
      batches.push_back(std::move(cur));
      cur = Batch{};
    }
  };
  for (size_t r = 0; r < prefix_len.size(); ++r) {
    const int64_t prefix = prefix_len[r];
    size_t item = 0;
    while (item < item_len[r].size()) {
      const int64_t tokens = item_len[r][item];
      if (prefix + tokens > max_batch_tokens)
        fail(SR_OVERSIZE_ITEM, "item " + std::to_string(item) + " needs " +
                                   std::to_string(prefix + tokens) + " tokens, over budget " +
                                   std::to_string(max_batch_tokens));
      const bool open = !cur.entries.empty() &&
                        cur.entries.back().request_index == static_cast<int32_t>(r) &&
                        cur.entries.back().item_end == static_cast<int32_t>(item);
      const int64_t cost = open ? tokens : prefix + tokens;
      if (cur.token_count + cost > max_batch_tokens) {
        flush();
        continue;
      }
      if (open)
        cur.entries.back().item_end = static_cast<int32_t>(item + 1);
      else
        cur.entries.push_back(
            {static_cast<int32_t>(r), static_cast<int32_t>(item), static_cast<int32_t>(item + 1)});
      cur.token_count += cost;
      ++item;
    }
  }
  flush();
  return batches;
}

std::vector<HostTopk> topk_host(const double* scores, const int64_t* ids, int32_t n, int32_t k) {
  std::vector<HostTopk> v(n);
  for (int32_t i = 0; i < n; ++i) v[i] = {scores[i], ids ? ids[i] : i, i};
  const int32_t kk = std::min(std::max(k, 0), n);
  std::partial_sort(v.begin(), v.begin() + kk, v.end(), [](const HostTopk& a, const HostTopk& b) {
    if (a.score != b.score) return a.score > b.score;
    if (a.id != b.id) return a.id < b.id;
    return a.index < b.index;
  });
  v.resize(kk);
  return v;
}

}  // namespace srh
