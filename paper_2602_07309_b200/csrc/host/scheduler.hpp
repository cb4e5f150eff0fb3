// Latency-bounded request scheduler: concurrent callers
// submit whole scoring requests; one dispatcher thread packs the queued ones
// into device passes (the engine's packed multi-request pass, one captured
// CUDA graph per pass shape) and completes each request's ticket.
//
// Reference behaviour this serves:
//   ScoringEngine::score serialises callers under one mutex (engine.cpp:389-392):
//     here callers never hold the engine; the dispatcher is its only user.
//   plan_batches packs requests FIFO under a token budget (engine.cpp:278-326):
//     the same greedy FIFO rule over whole requests (max_rows), plus a request
//     cap and a latency rule (below).
//   p50 / p99 are nearest-rank percentiles (service.cpp:28-34,
//     simulation.cpp:58-63): sorted[ceil(q*n) - 1].
//
// Batch formation when the device is free (FIFO, at least one request):
//   add the next queued request while
//     count < max_queries, rows + r.rows <= max_rows, and (budget_ms > 0)
//     age(oldest) + est_ms(rows + r.rows) <= budget_ms,
//   where est_ms(rows) = ms_per_row * rows is learned from the passes run so
//   far (EWMA). With max_wait_us > 0 an unfilled batch waits up to that long
//   after its oldest request's arrival for more arrivals. With sat_rows > 0 a
//   request of at least sat_rows rows runs in a pass of its own: it fills the
//   device alone, a bigger pass costs the same time per row, so batching it
//   would only lengthen the wait of the requests behind it. Smaller requests
//   batch as above (their passes amortise per-pass host work).
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "common.hpp"
#include "model.hpp"

namespace srh {

struct SchedOptions {
  int32_t max_queries = 8;
  int64_t max_rows = int64_t(1) << 22;
  double budget_ms = 0.0;   // 0 = no latency rule
  int32_t max_wait_us = 0;  // 0 = dispatch what is queued
  int32_t k = 10;
  bool borrow = false;  // inputs borrowed until wait() instead of copied at submit
  int64_t sat_rows = 0;  // requests of at least this many rows run alone (0 = off)
};

// A request deep-copied at submit (callers' buffers are borrowed per call).
struct OwnedRequest {
  std::vector<int32_t> prefix, offsets, tokens;
  std::vector<float> rows;
  std::vector<int64_t> ids;
  sr_request view{};
  int64_t n_rows = 0;  // packed rows: t_q + sum of item lengths
  void take(const sr_request& r, int32_t d_model, bool borrow);
};

struct Ticket {
  OwnedRequest req;
  std::vector<double> scores;
  std::vector<int64_t> top_ids;
  std::vector<double> top_scores;
  std::vector<int32_t> top_index;
  sr_result res{};
  int32_t status = SR_OK;
  std::string error;
  double t_submit = 0, t_start = 0, t_done = 0;  // ms, steady clock
  int32_t batch_queries = 0;
  bool done = false;
};

// Runs one pass over n packed requests (the engine, or a host stand-in in tests).
using SchedExec = std::function<void(const sr_request* reqs, int n, sr_result* res)>;

struct SchedStats {
  int64_t submitted = 0, completed = 0, failed = 0, batches = 0;
  double mean_batch = 0, p50_ms = 0, p99_ms = 0, max_ms = 0, mean_ms = 0;
  double ms_per_row = 0;  // current estimate
  double busy_ms = 0;     // sum of pass durations
  double max_pass_ms = 0; // longest pass
  double max_wait_ms = 0; // longest queue wait (submit -> pass start)
};

double percentile_nearest_rank(std::vector<double> v, double q);

class Scheduler {
 public:
  Scheduler(SchedExec exec, const ModelConfig& cfg, const SchedOptions& opt);
  ~Scheduler();
  Scheduler(const Scheduler&) = delete;
  Scheduler& operator=(const Scheduler&) = delete;

  // Validates (same categories as scoring) and queues; returns the ticket id.
  uint64_t submit(const sr_request& req);
  // Blocks until the ticket completes; copies scores / top-k into res (the
  // caller's buffers, as sr_engine_score) and releases the ticket. The
  // request's own failure is rethrown.
  void wait(uint64_t ticket, sr_result* res, double* latency_ms, int32_t* batch_queries);
  SchedStats stats(bool reset);

 private:
  void loop();
  double now_ms() const;

  SchedExec exec_;
  ModelConfig cfg_;
  SchedOptions opt_;
  std::mutex mu_;
  std::condition_variable cv_in_, cv_out_;
  std::deque<uint64_t> queue_;
  std::map<uint64_t, std::unique_ptr<Ticket>> tickets_;
  uint64_t next_ = 1;
  bool stop_ = false;
  double ms_per_row_ = 0;
  // stats since the last reset
  std::vector<double> lat_;
  std::vector<int32_t> batch_sizes_;
  int64_t submitted_ = 0, failed_ = 0;
  double busy_ms_ = 0;
  double max_pass_ms_ = 0;
  double max_wait_ms_ = 0;
  std::thread thread_;
};

}  // namespace srh
