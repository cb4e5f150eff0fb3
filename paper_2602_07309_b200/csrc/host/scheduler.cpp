// Latency-bounded request scheduler; see scheduler.hpp.
#include "scheduler.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>

#include "planner.hpp"

namespace srh {

double percentile_nearest_rank(std::vector<double> v, double q) {
  // service.cpp:28-34 percentile_of / simulation.cpp:58-63
  if (v.empty()) return 0;
  std::sort(v.begin(), v.end());
  const auto idx = static_cast<size_t>(std::ceil(q * static_cast<double>(v.size()))) - 1;
  return v[std::min(idx, v.size() - 1)];
}

void OwnedRequest::take(const sr_request& r, int32_t d_model, bool borrow) {
  n_rows = r.t_q + (r.n_items > 0 ? r.item_offsets[r.n_items] : 0);
  view = r;
  if (borrow) return;  // the caller keeps its arrays alive until wait()
  prefix.assign(r.prefix_tokens, r.prefix_tokens + std::max(r.t_q, 0));
  offsets.assign(r.item_offsets, r.item_offsets + r.n_items + 1);
  const int64_t total = offsets.back();
  if (r.mode == SR_MODE_MIXED) {
    rows.assign(r.item_rows, r.item_rows + total * d_model);
    tokens.clear();
  } else {
    tokens.assign(r.item_tokens, r.item_tokens + total);
    rows.clear();
  }
  if (r.item_ids)
    ids.assign(r.item_ids, r.item_ids + r.n_items);
  else
    ids.clear();
  view.prefix_tokens = prefix.data();
  view.item_offsets = offsets.data();
  view.item_tokens = tokens.empty() ? nullptr : tokens.data();
  view.item_rows = rows.empty() ? nullptr : rows.data();
  view.item_ids = ids.empty() ? nullptr : ids.data();
}

Scheduler::Scheduler(SchedExec exec, const ModelConfig& cfg, const SchedOptions& opt)
    : exec_(std::move(exec)), cfg_(cfg), opt_(opt) {
  if (opt_.max_queries < 1) fail(SR_PARAMETER, "scheduler max_queries must be >= 1");
  if (opt_.max_rows < 1) fail(SR_PARAMETER, "scheduler max_rows must be >= 1");
  if (opt_.budget_ms < 0 || opt_.max_wait_us < 0 || opt_.sat_rows < 0)
    fail(SR_PARAMETER, "scheduler budget and wait must be >= 0");
  if (opt_.k < 0 || opt_.k > 4096) fail(SR_PARAMETER, "top-k must be in [0, 4096]");
  thread_ = std::thread([this] { loop(); });
}

Scheduler::~Scheduler() {
  {
    std::lock_guard<std::mutex> lock(mu_);
    stop_ = true;
  }
  cv_in_.notify_all();
  if (thread_.joinable()) thread_.join();
  // tickets still queued fail; waiters (if any) are woken
  std::lock_guard<std::mutex> lock(mu_);
  for (auto& [id, t] : tickets_)
    if (!t->done) {
      t->status = SR_STATE_INVALID;
      t->error = "scheduler destroyed";
      t->done = true;
    }
  cv_out_.notify_all();
}

double Scheduler::now_ms() const {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

uint64_t Scheduler::submit(const sr_request& req) {
  if (req.n_items < 0 || (req.n_items > 0 && !req.item_offsets) || (req.t_q > 0 && !req.prefix_tokens))
    fail(SR_SPEC_VIOLATION, "null argument");
  validate_request(cfg_, req);  // the request's own error, at submit time
  auto t = std::make_unique<Ticket>();
  t->req.take(req, cfg_.d_model, opt_.borrow);
  const int32_t n = req.n_items, T = 1 + static_cast<int32_t>(cfg_.head_specs.size());
  const int32_t kk = std::max(opt_.k, 1);
  t->scores.assign(static_cast<size_t>(std::max(n, 1)) * T, 0.0);
  t->top_ids.assign(kk, 0);
  t->top_scores.assign(kk, 0.0);
  t->top_index.assign(kk, 0);
  t->res.scores = t->scores.data();
  t->res.k = opt_.k;
  t->res.topk_ids = t->top_ids.data();
  t->res.topk_scores = t->top_scores.data();
  t->res.topk_index = t->top_index.data();
  uint64_t id;
  {
    std::lock_guard<std::mutex> lock(mu_);
    if (stop_) fail(SR_STATE_INVALID, "scheduler stopped");
    id = next_++;
    t->t_submit = now_ms();
    tickets_[id] = std::move(t);
    queue_.push_back(id);
    ++submitted_;
  }
  cv_in_.notify_one();
  return id;
}

void Scheduler::wait(uint64_t id, sr_result* res, double* latency_ms, int32_t* batch_queries) {
  std::unique_ptr<Ticket> t;
  {
    std::unique_lock<std::mutex> lock(mu_);
    auto it = tickets_.find(id);
    if (it == tickets_.end()) fail(SR_PARAMETER, "unknown scheduler ticket");
    Ticket* p = it->second.get();
    cv_out_.wait(lock, [&] { return p->done; });
    t = std::move(it->second);
    tickets_.erase(it);
  }
  if (latency_ms) *latency_ms = t->t_done - t->t_submit;
  if (batch_queries) *batch_queries = t->batch_queries;
  if (t->status != SR_OK) fail(static_cast<sr_status>(t->status), t->error);
  if (!res) return;
  const int32_t n = t->req.view.n_items, T = 1 + static_cast<int32_t>(cfg_.head_specs.size());
  if (res->scores)
    std::memcpy(res->scores, t->scores.data(), static_cast<size_t>(n) * T * sizeof(double));
  const int32_t kr = std::min(std::max(res->k, 0), t->res.k_returned);
  for (int32_t j = 0; j < kr; ++j) {
    if (res->topk_ids) res->topk_ids[j] = t->top_ids[j];
    if (res->topk_scores) res->topk_scores[j] = t->top_scores[j];
    if (res->topk_index) res->topk_index[j] = t->top_index[j];
  }
  res->k_returned = kr;
  res->flops = t->res.flops;
  res->kv_incremental_per_item = t->res.kv_incremental_per_item;
}

SchedStats Scheduler::stats(bool reset) {
  std::lock_guard<std::mutex> lock(mu_);
  SchedStats s;
  s.submitted = submitted_;
  s.completed = static_cast<int64_t>(lat_.size());
  s.failed = failed_;
  s.batches = static_cast<int64_t>(batch_sizes_.size());
  double nb = 0;
  for (int32_t b : batch_sizes_) nb += b;
  s.mean_batch = batch_sizes_.empty() ? 0 : nb / batch_sizes_.size();
  s.p50_ms = percentile_nearest_rank(lat_, 0.50);
  s.p99_ms = percentile_nearest_rank(lat_, 0.99);
  double sum = 0, mx = 0;
  for (double v : lat_) {
    sum += v;
    mx = std::max(mx, v);
  }
  s.mean_ms = lat_.empty() ? 0 : sum / lat_.size();
  s.max_ms = mx;
  s.ms_per_row = ms_per_row_;
  s.busy_ms = busy_ms_;
  s.max_pass_ms = max_pass_ms_;
  s.max_wait_ms = max_wait_ms_;
  if (reset) {
    lat_.clear();
    batch_sizes_.clear();
    submitted_ = failed_ = 0;
    busy_ms_ = max_pass_ms_ = max_wait_ms_ = 0;
  }
  return s;
}

void Scheduler::loop() {
  std::vector<Ticket*> batch;
  std::vector<sr_request> reqs;
  std::vector<sr_result> res;
  for (;;) {
    batch.clear();
    {
      std::unique_lock<std::mutex> lock(mu_);
      cv_in_.wait(lock, [&] { return stop_ || !queue_.empty(); });
      if (stop_) return;
      for (;;) {
        // greedy FIFO under the request cap, the row budget and the latency rule
        const double now = now_ms();
        const double age = now - tickets_[queue_.front()]->t_submit;
        int64_t rows = 0;
        size_t take = 0;
        bool limited = false;
        for (uint64_t id : queue_) {
          const Ticket* t = tickets_[id].get();
          const int64_t r2 = rows + t->req.n_rows;
          // a request that fills the device alone (sat_rows) is never batched
          const bool alone = opt_.sat_rows > 0 && t->req.n_rows >= opt_.sat_rows;
          if (take > 0 && (static_cast<int32_t>(take) >= opt_.max_queries || r2 > opt_.max_rows ||
                           alone ||
                           (opt_.budget_ms > 0 && ms_per_row_ > 0 &&
                            age + ms_per_row_ * static_cast<double>(r2) > opt_.budget_ms))) {
            limited = true;
            break;
          }
          rows = r2;
          ++take;
          if (static_cast<int32_t>(take) >= opt_.max_queries || alone) {
            limited = true;
            break;
          }
        }
        const double wait_left = opt_.max_wait_us * 1e-3 - age;
        if (!limited && wait_left > 0) {
          // room left and the oldest request may still wait for company
          cv_in_.wait_for(lock, std::chrono::duration<double, std::milli>(wait_left),
                          [&] { return stop_ || queue_.size() > take; });
          if (stop_) return;
          if (queue_.size() > take) continue;  // re-form with the new arrivals
        }
        for (size_t i = 0; i < take; ++i) {
          batch.push_back(tickets_[queue_.front()].get());
          queue_.pop_front();
        }
        break;
      }
    }
    reqs.clear();
    res.clear();
    int64_t rows = 0;
    for (Ticket* t : batch) {
      reqs.push_back(t->req.view);
      res.push_back(t->res);
      rows += t->req.n_rows;
    }
    const double t0 = now_ms();
    int32_t status = SR_OK;
    std::string err;
    try {
      exec_(reqs.data(), static_cast<int>(reqs.size()), res.data());
    } catch (const Error& e) {
      status = e.code();
      err = e.what();
    } catch (const std::exception& e) {
      status = SR_CUDA;
      err = e.what();
    }
    const double t1 = now_ms();
    {
      std::lock_guard<std::mutex> lock(mu_);
      const double per_row = (t1 - t0) / static_cast<double>(std::max<int64_t>(rows, 1));
      if (status == SR_OK) ms_per_row_ = ms_per_row_ == 0 ? per_row : 0.7 * ms_per_row_ + 0.3 * per_row;
      busy_ms_ += t1 - t0;
      max_pass_ms_ = std::max(max_pass_ms_, t1 - t0);
      batch_sizes_.push_back(static_cast<int32_t>(batch.size()));
      for (size_t i = 0; i < batch.size(); ++i) {
        Ticket* t = batch[i];
        t->res = res[i];
        t->status = status;
        t->error = err;
        t->t_start = t0;
        t->t_done = t1;
        t->batch_queries = static_cast<int32_t>(batch.size());
        t->done = true;
        max_wait_ms_ = std::max(max_wait_ms_, t0 - t->t_submit);
        if (status == SR_OK)
          lat_.push_back(t1 - t->t_submit);
        else
          ++failed_;
      }
    }
    cv_out_.notify_all();
  }
}

}  // namespace srh
