#!/usr/bin/env python3
"""Benchmark: query-item pairs scored per second (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[1] — 0.6B-class pruned SLM (L20 d1024 H8
ff1536, V300, fan-in random init, seed 2026), 1 query x 256 candidates,
256-token shared prefix, 96-token item segments, synthetic uniform token ids.
A step = one full pass of the hot path over one query: packed shared-prefix
prefill through all 20 layers, final-LN score head, top-k.

Multi-GPU (torchrun, one rank per GPU): BASELINE.json configs[4] ("c5", the
default when WORLD_SIZE > 1) — 1 query x 8192 candidates of the C2 model split
contiguously across the ranks (global ids kept), prefix recomputed per rank,
per-rank top-k lists merged with one NCCL all-gather + device merge inside the
step (strong scaling). value = 8192 pairs / max-over-ranks time. At N=1 the
line carries the same C5 workload on one GPU under "c5".

  value : device-resident inputs, CUDA-graph replay + NCCL merge, CUDA events
          on the engine stream
  e2e   : the public API call ScoringEngine.score (ctypes -> C-ABI): host
          token arrays in, host scores + top-k out, every copy inside the step

--impl reference times the reference's own CPU implementation
(oracle/_ref: reference sources compiled in place; else the C port) on
bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (n_layers, d_model, n_heads, d_ff, t_q, t_i, n_items per GPU, soft_tokens)
    "c2": (20, 1024, 8, 1536, 256, 96, 256, False),
    "c3": (20, 1024, 8, 1536, 256, 8, 1024, True),
    "c3_rows": (20, 1024, 8, 1536, 256, 8, 1024, True),
    "c1": (2, 64, 4, 256, 500, 50, 64, False),
    "c4": (28, 2048, 16, 6144, 256, 96, 250, False),
    # configs[4]: 8192 candidates in total, split across the ranks (strong scaling)
    "c5": (20, 1024, 8, 1536, 256, 96, 8192, False),
}
STRONG = {"c5"}  # n_items is the whole job's, not per GPU
# configs[2] context compression: items arrive as compact d_emb embeddings and
# are projected on the device into t_i soft-token rows (sr_engine_set_projection;
# SURVEY H7, north_star (d)). "c3_rows" sends the d_model-wide rows instead.
EMB = {"c3": 256}
SERVE_WORKLOADS = {"c2", "c4", "c3_rows"}  # served through sr_sched_* (c3_rows: soft rows)
# queries packed into one device pass per step (per GPU)
QUERIES = {"c4": 32}
WORKLOAD_DESC = {
    "c4": "1.7B-class unpruned teacher-shaped ranker (L28 d2048 H16 ff6144), 32 queries x 250 "
          "candidates per step in one packed pass, 256-token prefixes, 96-token items",
    "c2": "0.6B-class pruned SLM (L20 d1024 H8 ff1536), 1 query x 256 candidates, "
          "256-token shared prefix, 96-token items",
    "c3": "0.6B-class pruned SLM, 1 query x 1024 candidates, 256-token prefix, items as "
          "256-d embeddings projected on the device into 8 soft-token rows (context compression)",
    "c3_rows": "0.6B-class pruned SLM, 1 query x 1024 candidates, 256-token prefix, "
          "8 soft-token rows per item (context compression)",
    "c1": "reference default toy ranker (L2 d64 H4 ff256), 1 query x 64 candidates, "
          "T_q 500, T_i 50 (cmd_bench shape)",
    "c5": "candidate-sharded ranking: 1 query x 8192 candidates (C2 model, 96-token items, "
          "256-token prefix) split across the GPUs, NCCL top-k merge",
}


def shard(wl, world, rank):
    """(items on this rank, global id of its first item, items in the whole job)."""
    n = WORKLOADS[wl][6]
    if wl in STRONG:
        base, extra = divmod(n, world)
        n_loc = base + (1 if rank < extra else 0)
        lo = rank * base + min(rank, extra)
        return n_loc, lo, n
    return n, rank * n, n * world


def config_for(wl, world):
    """The workload description both arms print (identical dicts)."""
    L, d, H, ff, t_q, t_i, n, soft = WORKLOADS[wl]
    nq = QUERIES.get(wl, 1)
    _, _, n_all = shard(wl, world, 0)
    par = ("single-gpu" if world == 1 else f"query-batch replicas x{world}" if nq > 1 else
           f"candidate-shard x{world}")
    return {"workload": WORKLOAD_DESC[wl], "model": f"semrank-{wl}-L{L}-d{d}",
            "global_batch": n_all * nq, "seq_len": t_q + t_i, "queries_per_step": nq * (
                world if wl not in STRONG and nq > 1 else 1),
            "candidates_per_query": n_all if wl in STRONG else n * (world if nq == 1 else 1),
            "parallelism": par, "top_k": TOPK,
            "l2": "inputs+weights+activations per step > 126 MB L2 (no flush)"}
TOPK = 10  # service page size (service.hpp:24)


def model_flops_per_query(L, d, ff, t_q, lens):
    """linear 2L(T)(4d^2+2d ff) + attention 4dL[pairs] + head."""
    T = t_q + sum(lens)
    lin = 2.0 * L * T * (4 * d * d + 2 * d * ff)
    pairs = t_q * (t_q + 1) / 2 + sum(t_q * l + l * (l + 1) / 2 for l in lens)
    att = 4.0 * d * L * pairs
    return lin, att, 2.0 * d * 7 * len(lens)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def load_traffic():
    """dram bytes per GEMM launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.path = tempfile.mktemp(prefix="clk_", suffix=".csv")
        self.proc = None
        self.gpu = gpu_index

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                p = [x.strip() for x in line.split(",")]
                if len(p) < 9:
                    continue
                try:
                    sm.append(float(p[1]))
                    smax = float(p[2])
                except ValueError:
                    continue
                for n, v in zip(names, p[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        os.unlink(self.path)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_request(sr, wl, world, rank, seed=7):
    L, d, H, ff, t_q, t_i, _, soft = WORKLOADS[wl]
    rng = np.random.default_rng(seed)
    prefix = rng.integers(0, 256, t_q).astype(np.int32)
    n_loc, lo, n_all = shard(wl, world, rank)
    req = sr.ScoreRequest(request_id=f"bench-{wl}", prefix_tokens=prefix,
                          mode=sr.ScoreMode.Mixed if soft else sr.ScoreMode.MultiItem)
    if soft:
        # soft-token rows ~ N(0, 0.08^2) (the reference's embedding scale)
        rows = rng.standard_normal((n_all, t_i, d)).astype(np.float32) * np.float32(0.08)
        for i in range(lo, lo + n_loc):
            req.items.append(sr.ScoreItem(id=str(i), embedding=rows[i], n_emb_tokens=t_i))
    else:
        toks = rng.integers(0, 256, (n_all, t_i)).astype(np.int32)
        for i in range(lo, lo + n_loc):
            req.items.append(sr.ScoreItem(id=str(i), tokens=toks[i]))
    ids = np.arange(lo, lo + n_loc, dtype=np.int64)
    return req, ids


def make_queries(sr, wl, n_queries, rank):
    """n_queries independent requests (own prefixes and items) for batched workloads."""
    out = []
    for q in range(n_queries):
        req, _ = make_request(sr, wl, 1, 0, seed=1000 * (rank + 1) + q)
        req.request_id = f"bench-{wl}-{q}"
        out.append(req)
    return out


# ------------------------------------------------------------- CPU baseline
class _RefCfg:
    """ModelConfig fields the oracle harness reads (the reference arm never
    imports the product)."""

    class _Head:
        def __init__(self, name):
            self.name, self.arity = name, 1

    def __init__(self, wl):
        L, d, H, ff = WORKLOADS[wl][:4]
        self.n_layers, self.d_model, self.n_heads, self.d_ff = L, d, H, ff
        self.vocab_size, self.max_seq, self.yes_token_id, self.no_token_id = 300, 4096, 261, 262
        self.head_specs = [self._Head(n) for n in ("click", "apply", "badfit", "shortlist",
                                                   "dismiss")]


def reference_weights(wl):
    """SRNKWTS1 file of the workload's weights written by the reference's own
    Rng + save_weights (oracle/_ref), else by the C port — byte-identical to
    the product's init_model (tests/test_host.py). Test infrastructure only."""
    from oracle import oracle as O
    fd, path = tempfile.mkstemp(prefix=f"bench_{wl}_", suffix=".srnk")
    os.close(fd)
    fan_in = wl != "c1"
    seed = 2026 if fan_in else 1
    cfg = _RefCfg(wl)
    if O.ref_available():
        O.ref_init_save(cfg, seed, path, fan_in=fan_in)
    else:
        O.OracleWeights.init(cfg, seed, 1 if fan_in else 0).save(path)
    return path


def cpu_reference_run(wl, n_items, weights_path, threads):
    """One query on the host: prefix + the first n_items items of the
    workload's request stream, reference multi_item (tokens) or mixed (soft
    rows) mode; returns (seconds, kind). Test infrastructure only."""
    from oracle import oracle as O
    L, d, H, ff, t_q, t_i, _, soft = WORKLOADS[wl]
    rng = np.random.default_rng(7)
    prefix = rng.integers(0, 256, t_q).astype(np.int32)
    if soft:
        rows = [rng.standard_normal((t_i, d)).astype(np.float32) * np.float32(0.08)
                for _ in range(n_items)]
        items = None
    else:
        items = [rng.integers(0, 256, t_i).astype(np.int32) for _ in range(n_items)]
        rows = None
    if O.ref_available():
        O.ref().ref_set_parallel(1)
        t0 = time.perf_counter()
        O.ref_score(weights_path, 3 if soft else 2, prefix, items=items, rows=rows)
        return time.perf_counter() - t0, "reference"
    w = O.OracleWeights.load(weights_path)
    t0 = time.perf_counter()
    w.score(prefix, items=items, rows=rows, threads=threads)
    return time.perf_counter() - t0, "port"


SAMPLE_ITEMS = {"c1": 64, "c2": 8, "c3": 48, "c3_rows": 48, "c4": 3, "c5": 8}


def reference_query_time(wl, path, threads):
    """One bounded sample of one query of the workload on the host.

    Runs the reference on (prefix + 1 item) and (prefix + S items) and fits its
    cost model t(n) = a + n b (a = prefix prefill, b = one item). The reference
    scores a whole query of N items as score_multi_item_chunked does
    (engine.cpp:328-377): greedy chunks under max_seq, each chunk repaying the
    prefix — or, in mixed mode, score_mixed's single prefix (engine.cpp:238-276)
    — so one query costs chunks(N) a + N b. Returns (seconds per query, kind,
    detail)."""
    L, d, H, ff, t_q, t_i, n, soft = WORKLOADS[wl]
    n_q = n  # items of one query (C5: the whole 8192)
    S = min(SAMPLE_ITEMS.get(wl, 8), n_q)
    t1, kind = cpu_reference_run(wl, 1, path, threads)
    if S == n_q and (soft or t_q + n_q * t_i <= 4096):
        tS, kind = cpu_reference_run(wl, S, path, threads)
        return tS, kind, f"full query ({n_q} items) {tS:.2f} s"
    tS, kind = cpu_reference_run(wl, S, path, threads)
    b = max(tS - t1, 0.0) / (S - 1)
    a = max(t1 - b, 0.0)
    per_chunk = max(1, (4096 - t_q) // t_i)
    chunks = 1 if soft else -(-n_q // per_chunk)
    return chunks * a + n_q * b, kind, (f"t(1 item) {t1:.2f} s, t({S} items) {tS:.2f} s -> "
                                        f"a {a:.3f} s, b {b:.4f} s, {chunks} chunk(s)")


def cpu_baseline(wl, samples=3):
    """The reference CPU path on the box's host cores (rank 0, N=1 only)."""
    L, d, H, ff, t_q, t_i, n, soft = WORKLOADS[wl]
    nq = QUERIES.get(wl, 1)
    path = reference_weights(wl)
    threads = os.cpu_count() or 1
    try:
        cpu_reference_run(wl, 1, path, threads)  # loads + caches the weights (not timed)
        ts = []
        for _ in range(samples):
            tq, kind, detail = reference_query_time(wl, path, threads)
            ts.append(tq)
    finally:
        os.unlink(path)
    tq = statistics.median(ts)
    return {"value": n / tq, "unit": "pairs/s", "cores": threads, "kind": kind,
            "sample": _sample_text(wl, detail, samples) + (f"; x{nq} queries per step"
                                                           if nq > 1 else "")}


def _sample_text(wl, detail, samples):
    L, d, H, ff, t_q, t_i, n, soft = WORKLOADS[wl]
    mode = "score_mixed" if soft else "score_multi_item_chunked"
    return (f"per sample: the reference ({mode}, OpenMP on all host threads) on the prefix + 1 "
            f"and + S items of the workload's first query, extrapolated with its own cost "
            f"model chunks(N)*prefix + N*item to the full {n}-item query; median of {samples}: "
            f"{detail}")


# ---------------------------------------------------------------- main arms
def run_reference_arm(args):
    """The reference's own CPU implementation (oracle/_ref) on the same
    workload, config and metric as our arm; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    wl = args.workload
    L, d, H, ff, t_q, t_i, n, soft = WORKLOADS[wl]
    nq = QUERIES.get(wl, 1)
    _, _, n_all = shard(wl, world, 0)
    queries = nq * (world if wl not in STRONG else 1) if nq > 1 else 1
    path = reference_weights(wl)
    threads = os.cpu_count() or 1
    times, detail, kind = [], "", "reference"
    try:
        for s_ in range(args.warmup + args.steps):
            tq, kind, detail = reference_query_time(wl, path, threads)
            if s_ >= args.warmup:
                times.append(tq * queries if nq > 1 else tq * (n_all / n))
    finally:
        os.unlink(path)
    pairs = n_all * nq if nq > 1 else n_all
    value = pairs * len(times) / sum(times)
    sample = _sample_text(wl, detail, args.steps)
    line = {"metric": "query-item pairs scored/sec", "value": value, "unit": "pairs/s",
            "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * statistics.mean(times), "higher_is_better": True,
            "scaling": "strong" if wl in STRONG else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": config_for(wl, world),
            "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": kind,
                             "sample": sample},
            "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SR_BENCH_COMM=host (test aid): ranks exchange their top-k through the
    # product's host-transport communicator over gloo, so the N > 1 path can be
    # exercised with several ranks on one GPU (NCCL refuses that).
    host_comm = os.environ.get("SR_BENCH_COMM") == "host"
    if host_comm:
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if host_comm:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2602_07309_b200 as sr

    wl = args.workload
    L, d, H, ff, t_q, t_i, _, soft = WORKLOADS[wl]
    n_loc, _, n_all = shard(wl, world, rank)
    cfg = sr.ModelConfig(n_layers=L, d_model=d, n_heads=H, d_ff=ff,
                         head_specs=sr.ModelConfig.default_toy().head_specs)
    weights = sr.init_model(cfg, 2026 if wl != "c1" else 1, "fan_in" if wl != "c1" else "reference")
    eng = sr.ScoringEngine(weights, device=local)
    nq = QUERIES.get(wl, 1)
    k = TOPK
    comm = None
    reqs = None
    if nq > 1:
        # batched queries: independent per rank (replicas), one packed pass per step
        reqs = make_queries(sr, wl, nq, rank)
        req, ids = reqs[0], None
        plan = sr.BatchPlan(eng, reqs, k)
    elif wl in EMB:
        # compact embeddings in, projection to soft rows inside the device pass
        req, ids = None, None
        rng = np.random.default_rng(7)
        prefix = rng.integers(0, 256, t_q).astype(np.int32)
        emb = rng.standard_normal((n_loc, EMB[wl])).astype(np.float32)
        proj = (np.random.default_rng(2027).standard_normal((EMB[wl], t_i * d))
                * (0.08 / np.sqrt(EMB[wl]))).astype(np.float32)
        eng.set_projection(proj, t_i)
        plan = eng.plan_embeddings(prefix, emb, "project", k=k)
    else:
        req, ids = make_request(sr, wl, world, rank)
        if world > 1 and host_comm:
            def allgather(b):
                out = [None] * world
                dist.all_gather_object(out, b)
                return out
            comm = sr.Comm.host(world, rank, local, allgather)
        elif world > 1:
            uid = sr.Comm.unique_id() if rank == 0 else bytes(128)
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            comm = sr.Comm(world, rank, obj[0], local)
        plan = eng.plan(req, k=k, item_ids=ids)
    stream = torch.cuda.ExternalStream(eng.stream_ptr)

    def step():
        if comm is not None:
            plan.run_sharded(comm)
        else:
            plan.run()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    plan.sync()

    # -------------------------------------------------- device-resident value
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for i in range(args.steps):
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    plan.sync()
    barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = ev[0][0].elapsed_time(ev[-1][1])
    t = torch.tensor([total_ms], device="cuda")
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    pairs = n_all * nq * args.steps  # the whole job's pairs (all ranks)
    value = pairs / (total_ms / 1000.0)
    lat_sorted = sorted(step_ms)
    p99 = lat_sorted[max(0, int(np.ceil(0.99 * len(lat_sorted))) - 1)]  # service.cpp:28-34
    result = plan.fetch_all()[0] if nq > 1 else plan.fetch()

    # ----------------------------------------------------------- e2e (public API)
    shape = plan.shape()

    def e2e_call():
        if nq > 1:
            eng.score_batch(reqs, k)
        elif wl in EMB:
            eng.score_embeddings(prefix, emb, "project", k=k)
        elif comm is not None:
            eng.score_sharded(comm, req, k, ids)
        else:
            eng.score(req, k)

    for _ in range(max(1, args.warmup)):
        e2e_call()
    barrier()
    e2e_times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        e2e_call()
        e2e_times.append(time.perf_counter() - t0)
    barrier()
    te = torch.tensor([sum(e2e_times)], device="cuda")
    if dist is not None:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = pairs / float(te.item())
    h2d = shape["h2d_bytes"]  # packed rows/spans/tiles/ids (+ soft rows), per call
    d2h = shape["d2h_bytes"]  # scores [N x tasks] f64 + top-k entries

    # -------------------------------------------------- per-kernel roofline
    prof = plan.profile(reps=3)
    lens = [t_i] * n_loc
    lin, att, head = (nq * v for v in model_flops_per_query(L, d, ff, t_q, lens))

    # latency-bounded throughput sweep over queries per pass (batched workloads)
    sweep = []
    if nq > 1:
        for b in sorted({1, max(1, nq // 4), nq}):
            bp = sr.BatchPlan(eng, reqs[:b], k)
            bp.run()
            bp.sync()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(3):
                bp.run()
            e1.record(stream)
            bp.sync()
            ms = e0.elapsed_time(e1) / 3
            sweep.append({"queries_per_pass": b, "latency_ms": round(ms, 3),
                          "pairs_per_s": round(b * n_loc / (ms / 1000.0), 1),
                          "meets_500ms": ms <= 500})
            del bp
    gemm_ms = sum(prof[c][0] for c in ("gemm_qkv", "gemm_o", "gemm_in", "gemm_out"))
    gemm_launches = sum(prof[c][1] for c in ("gemm_qkv", "gemm_o", "gemm_in", "gemm_out"))
    peaks, peak_kind = load_peaks()
    achieved = lin / (gemm_ms / 1000.0) / 1e12
    peak = peaks.get("bf16_tflops_sustained", 1391.8)
    traffic = load_traffic().get(f"{wl}_gemm_dram_bytes_per_launch")
    M = shape["rows"]
    attn_bytes = 8.0 * d * M * L  # §8(d): read Q,K,V + write O, bf16, per layer
    attn_ms = prof["attention"][0]
    roofline = {"bound": "tensor", "kernel": "tcgen05 GEMMs (QKV/O/W_in/W_out)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic,
                "peak_source": f"{peak_kind} bf16_tflops_sustained",
                "algorithmic_flops_per_launch": lin / max(gemm_launches, 1),
                "gemm_share_of_step": gemm_ms / max(sum(v[0] for v in prof.values()), 1e-9),
                "attention": {"bound": "hbm", "achieved_gbs": attn_bytes / (attn_ms / 1000) / 1e9,
                              "peak_gbs": peaks.get("hbm_gbs"),
                              "frac": attn_bytes / (attn_ms / 1000) / 1e9 / peaks.get("hbm_gbs", 1),
                              "achieved_tflops": att / (attn_ms / 1000) / 1e12},
                "per_class_ms": {c: round(v[0], 4) for c, v in prof.items()}}

    # configs[4] on this one GPU (the N=1 point of the C5 scaling curve)
    launches = plan.kernel_count() * args.steps
    serving = None
    if world == 1 and not args.no_serving and wl in SERVE_WORKLOADS:
        serving = serving_sweep(sr, eng, wl, total_ms / args.steps / nq)
    c5 = None
    if wl == "c2" and world == 1 and not args.no_c5:
        del plan
        c5 = c5_single_gpu(sr, eng, torch, stream)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(wl)
        except Exception as e:  # oracle missing on the box -> reported, not fatal
            cpu = {"value": None, "unit": "pairs/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"unavailable: {e}"}

    line = {
        "metric": "query-item pairs scored/sec", "value": value, "unit": "pairs/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if wl in STRONG else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": config_for(wl, world),
        "device_pass": {"tokens_per_pass_per_gpu": M, "items_per_gpu": n_loc,
                        "prefill_tokens_per_s_per_gpu": M / (total_ms / args.steps / 1000.0),
                        "p99_pass_ms": p99, "p50_pass_ms": statistics.median(step_ms),
                        "sweep": sweep or None},
        "e2e": {"value": e2e_value, "unit": "pairs/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "path": ("ScoringEngine.score_batch -> sr_engine_score_batch" if nq > 1 else
                         ("ScoringEngine.score_sharded -> sr_engine_score_sharded (" + ("host-transport" if host_comm else "NCCL") + " merge)")
                         if comm is not None else
                         "ScoringEngine.score_embeddings -> sr_engine_score_emb (projection on "
                         "the device)" if wl in EMB else
                         "ScoringEngine.score -> sr_engine_score") + " (host arrays in/out)"},
        "gpu_launches": launches,
        "clocks": clk, "roofline": roofline, "cpu_baseline": cpu, "c5": c5,
        "serving": serving,
        "topk_head": [(iid, round(s, 6)) for iid, s in result.topk[:3]],
    }
    ok = [p for p in sweep if p["meets_500ms"]]
    if ok:
        # batched workloads (configs[3]): the metric is pairs/s at a fixed p99
        # query latency, so the headline is the fastest pass size whose pass
        # time (every query's latency) is within 500 ms; the full-batch pass
        # stays under device_pass
        best = max(ok, key=lambda p: p["pairs_per_s"])
        line["value_basis"] = (f"best pass size meeting the 500 ms query latency: "
                               f"{best['queries_per_pass']} queries/pass at {best['latency_ms']} ms; "
                               f"full {nq}-query pass {total_ms / args.steps:.1f} ms")
        line["value"] = best["pairs_per_s"]
        line["ms_per_step"] = best["latency_ms"]
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def c5_single_gpu(sr, eng, torch, stream, steps=3, warmup=2):
    """BASELINE configs[4] (8192 candidates, C2 model) on one GPU: the N=1
    point of the strong-scaling curve the torchrun runs print as their value."""
    req, ids = make_request(sr, "c5", 1, 0)
    plan = eng.plan(req, k=TOPK, item_ids=ids)
    for _ in range(warmup):
        plan.run()
    plan.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        plan.run()
    e1.record(stream)
    plan.sync()
    ms = e0.elapsed_time(e1) / steps
    res = plan.fetch()
    out = {"workload": WORKLOAD_DESC["c5"] + " (1 GPU)", "value": 8192 / (ms / 1000.0),
           "unit": "pairs/s", "ms_per_step": ms, "steps": steps, "warmup": warmup,
           "gpu_launches": plan.kernel_count() * steps,
           "topk_head": [(iid, round(s, 6)) for iid, s in res.topk[:3]]}
    del plan
    return out


SERVE_BUDGETS_MS = (50.0, 500.0)  # p99 targets: interactive, and the paper's 500 ms
SERVE_LOADS = (0.3, 0.4, 0.5, 0.6, 0.7, 0.85, 0.95, 1.05)  # offered load, fraction of the 1-query pass rate
# Requests of at least this many packed rows run alone: one C2 / C4 request
# (~24.8k rows) already fills the GPU's GEMM waves, so batching it adds
# latency and no throughput; C3 requests (8.4k rows) batch as before.
SERVE_SAT_ROWS = 16384


def serving_sweep(sr, eng, wl, pass_ms, seconds=3.0, max_queries=8):
    """Pairs/s at a fixed p99 (BASELINE.json metric) through the native
    scheduler (sr_sched_*): open-loop Poisson arrivals of
    whole requests of the workload (host arrays, distinct prefixes and items),
    latency = submit -> completion on the host clock (queueing, H2D, device
    pass, D2H), p99 by nearest rank (service.cpp:28-34). For each budget the
    offered load is swept as a fraction of the 1-query device pass rate; the
    reported point is the highest-throughput load that the server sustained
    (completions kept pace: achieved >= 0.97 x offered queries/s, so an
    overloaded run whose queue is still growing never counts) and whose p99
    meets the budget."""
    import threading
    pool = make_queries(sr, wl, max_queries, rank=7)
    n_items = len(pool[0].items)
    # the largest pass's workspace first (a later growth would invalidate the
    # captured graphs), then every pass shape the scheduler can form, captured
    # before timing
    eng.reserve(sum(len(r.prefix_tokens) + sum(len(it.tokens) or it.n_emb_tokens for it in r.items)
                    for r in pool))
    for b in range(max_queries, 0, -1):
        eng.score_batch(pool[:b], TOPK)
    cap_qps = 1000.0 / pass_ms
    rng = np.random.default_rng(2027)
    out = {"arrivals": "open-loop Poisson, whole requests (host arrays) into sr_sched_submit",
           "latency": "submit -> completion, host clock; p99 nearest rank (service.cpp:28-34)",
           "pass_capacity_qps": cap_qps, "max_queries_per_pass": max_queries,
           "sat_rows": SERVE_SAT_ROWS, "budgets": {}}
    for budget in SERVE_BUDGETS_MS:
        points, best = [], None
        with sr.Scheduler(eng, k=TOPK, max_queries=max_queries, budget_ms=budget,
                          sat_rows=SERVE_SAT_ROWS) as s:
            packed = [s.pack(r) for r in pool]
            for j in range(3):  # learn the pass time
                s.wait(s.submit(pool[j % len(pool)], packed[j % len(pool)]))
            s.stats(reset=True)
            for frac in SERVE_LOADS:
                rate = frac * cap_qps
                # enough arrivals that the drain after the last one (about one
                # latency) stays small against the window: >= 300 queries (p99 = the 4th largest),
                # at most 12 s per point (slow passes, e.g. C4 at 50 ms)
                n = max(40, int(rate * min(12.0, max(seconds, 300.0 / rate))))
                gaps = rng.exponential(1.0 / rate, n)
                tickets, done = [], threading.Event()
                lock = threading.Condition()

                def waiter():
                    got = 0
                    while got < n:
                        with lock:
                            while len(tickets) <= got:
                                lock.wait()
                            t = tickets[got]
                        s.wait(t)
                        got += 1
                    done.set()

                th = threading.Thread(target=waiter)
                th.start()
                t0 = time.perf_counter()
                due = t0
                for j in range(n):
                    due += gaps[j]
                    while True:
                        left = due - time.perf_counter()
                        if left <= 0:
                            break
                        time.sleep(min(left, 0.002) if left > 0.0005 else 0)
                    q = j % len(pool)
                    t = s.submit(pool[q], packed[q])
                    with lock:
                        tickets.append(t)
                        lock.notify()
                done.wait()
                elapsed = time.perf_counter() - t0
                th.join()
                st = s.stats(reset=True)
                achieved_qps = n / elapsed
                pt = {"offered_load": frac, "offered_qps": round(rate, 2), "queries": n,
                      "achieved_qps": round(achieved_qps, 2),
                      "sustained": achieved_qps >= 0.97 * (n / (float(np.sum(gaps)) or 1e-9)),
                      "pairs_per_s": round(n * n_items / elapsed, 1),
                      "p50_ms": round(st["p50_ms"], 3), "p99_ms": round(st["p99_ms"], 3),
                      "max_ms": round(st["max_ms"], 3), "mean_ms": round(st["mean_ms"], 3),
                      "mean_pass_ms": round(st["busy_ms"] / max(st["batches"], 1), 3),
                      "max_pass_ms": round(st["max_pass_ms"], 3),
                      "max_wait_ms": round(st["max_wait_ms"], 3),
                      "mean_queries_per_pass": round(st["mean_batch"], 2),
                      "meets_budget": st["p99_ms"] <= budget}
                points.append(pt)
                if (pt["meets_budget"] and pt["sustained"]
                        and (best is None or pt["pairs_per_s"] > best["pairs_per_s"])):
                    best = pt
        out["budgets"][f"p99<={int(budget)}ms"] = {
            "pairs_per_s": best["pairs_per_s"] if best else None,
            "p99_ms": best["p99_ms"] if best else None,
            "offered_load": best["offered_load"] if best else None, "sweep": points}
    return out


# ------------------------------------------------ retrieval scan (§8(f) row 4)
RETRIEVAL = {
    # name: (docs per GPU, d_emb, features, k) — bench_kernels.cpp:130-164 shape,
    # and a production-scale corpus that exercises the HBM roofline
    "retrieval": (200_000, 32, 1, 100),
    "retrieval_xl": (33_554_432, 32, 1, 100),
}


def make_corpus(n, d, f, seed=7):
    rng = np.random.default_rng(seed)
    emb = np.empty((n, d), np.float32)
    step = 1 << 22
    for lo in range(0, n, step):  # bounded temporaries for the large corpus
        x = rng.standard_normal((min(step, n - lo), d), dtype=np.float32)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        emb[lo:lo + len(x)] = x
    feat = rng.random((n, f), dtype=np.float32)
    return emb, feat, np.arange(n, dtype=np.int64)


def run_retrieval(args):
    """docs scanned/s of exhaustive_topk (retrieval.cpp:134-173) through the
    public API (host query in, host top-K out; corpus resident in HBM)."""
    import paper_2602_07309_b200 as sr
    from paper_2602_07309_b200.retrieval import DeviceCorpus
    n, d, f, k = RETRIEVAL[args.workload]
    emb, feat, ids = make_corpus(n, d, f)
    corpus = DeviceCorpus(emb, feat, ids)
    rng = np.random.default_rng(11)
    queries = [emb[int(i)].copy() for i in rng.integers(0, n, args.warmup + args.steps)]
    w = [0.25]
    for q in queries[:args.warmup]:
        corpus.topk(q, 1.0, w, k)
    clk = ClockSampler(0)
    clk.start()
    times, scans = [], []
    for q in queries[args.warmup:]:
        t0 = time.perf_counter()
        got_ids, got_sc = corpus.topk(q, 1.0, w, k)
        times.append(time.perf_counter() - t0)
        scans.append(corpus.last_scan_ms())
    clocks = clk.stop()
    per_q = statistics.median(times)
    scan_ms = statistics.median(scans)
    bytes_per_doc = 4 * d + 4 * f  # algorithmic: embedding + features read once
    peaks, peak_kind = load_peaks()
    achieved = n * bytes_per_doc / (scan_ms / 1000.0) / 1e9
    cpu = None
    if not args.no_cpu_baseline:
        cpu = retrieval_cpu_baseline(emb, feat, ids, queries[-1], w, k)
    line = {"metric": "docs scanned/sec (exhaustive filtered top-K retrieval)",
            "value": n / per_q, "unit": "docs/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_q * 1000, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 scan + f64 rescore",
            "data": "synthetic (unit N(0,1) embeddings, U(0,1) feature)",
            "config": {"workload": f"{n} docs x d_emb {d}, {f} feature, k {k}, one query per "
                                   "step, no filter (bench_kernels.cpp:130-164 shape"
                                   + (")" if n == 200_000 else ", production-scale corpus)"),
                       "corpus_bytes": n * bytes_per_doc,
                       "l2": "corpus > L2" if n * bytes_per_doc > 126e6 else "corpus fits in L2"},
            "e2e": {"value": n / per_q, "unit": "docs/s", "h2d_bytes_per_step": 4 * d + 8 * f,
                    "d2h_bytes_per_step": 16 * k + 8,
                    "path": "DeviceCorpus.topk -> sr_corpus_topk (host query in, host top-K out)"},
            "gpu_launches": 4 * args.steps, "clocks": clocks,
            "roofline": {"bound": "hbm", "kernel": "retrieval_scan_bulk_kernel (fp32 TMA-streamed pass)",
                         "achieved": achieved, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                         "frac": achieved / peaks.get("hbm_gbs", 1.0),
                         "traffic": load_traffic().get(f"{args.workload}_scan_dram_bytes_per_launch"),
                         "peak_source": f"{peak_kind} hbm_gbs",
                         "algorithmic_bytes_per_launch": n * bytes_per_doc,
                         "scan_ms": scan_ms, "candidates_rescored": corpus.last_candidates()},
            "cpu_baseline": cpu, "topk_head": [(int(i), float(s)) for i, s in
                                               zip(got_ids[:3], got_sc[:3])]}
    print(json.dumps(line), flush=True)
    return 0


def retrieval_cpu_baseline(emb, feat, ids, q, w, k, budget_docs=2_000_000):
    """The reference's exhaustive_topk (oracle/_ref, OpenMP lane) on a bounded
    prefix of the corpus; else the C restatement. Test infrastructure only."""
    from oracle import oracle as O
    n = min(len(emb), budget_docs)
    threads = os.cpu_count() or 1
    if O.ref_available():
        O.ref().ref_set_parallel(1)
        secs = np.zeros(1)
        O.ref_topk(emb[:n], feat[:n], ids[:n], None, q, 1.0, w, None, k, timing=secs)
        t, kind = float(secs[0]), "reference"
    else:
        t0 = time.perf_counter()
        O.oracle_topk(emb[:n], feat[:n], ids[:n], None, q, 1.0, w, k)
        t, kind, threads = time.perf_counter() - t0, "port", 1
    return {"value": n / t, "unit": "docs/s", "cores": threads, "kind": kind,
            "sample": f"one query over the first {n} docs, exhaustive_topk call only "
                      f"(Exec::Parallel lane), {t:.3f} s"}


# ------------------------------------------------- /score wire ingest (§8(f) 2)
def run_wire(args):
    """C3 through the /score wire format: a JSON body whose 1024 items carry
    8 x 1024 float32 rows as embedding_b64 (service.cpp:361-370); per step
    parse_score_request_json + ScoringEngine.score (base64 decoded in HBM)."""
    import base64 as b64
    import torch
    import paper_2602_07309_b200 as sr
    L, d, H, ff, t_q, t_i, n_loc, soft = WORKLOADS["c3"]
    cfg = sr.ModelConfig(n_layers=L, d_model=d, n_heads=H, d_ff=ff,
                         head_specs=sr.ModelConfig.default_toy().head_specs)
    eng = sr.ScoringEngine(sr.init_model(cfg, 2026, "fan_in"), device=0)
    rng = np.random.default_rng(7)
    rows = rng.standard_normal((n_loc, t_i, d)).astype(np.float32) * np.float32(0.08)
    payloads = [b64.b64encode(rows[i].tobytes()).decode() for i in range(n_loc)]
    body = json.dumps({"request_id": "wire", "prefix_tokens": rng.integers(0, 256, t_q).tolist(),
                       "mode": "mixed", "items": [{"id": str(i), "embedding_b64": p}
                                                  for i, p in enumerate(payloads)]})
    raw = body.encode()
    for _ in range(args.warmup):
        eng.score_json(raw, k=TOPK)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = eng.score_json(raw, k=TOPK)  # native parse + device base64 decode + scoring
        times.append(time.perf_counter() - t0)
    per_q = statistics.median(times)
    t0 = time.perf_counter()
    eng.score(sr.parse_score_request_json(body, d), k=TOPK)  # Python json mirror, for contrast
    py_ms = (time.perf_counter() - t0) * 1000
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import oracle as O
        if O.ref_available():
            t0 = time.perf_counter()
            for p in payloads:
                O.ref_decode_f32_base64(p)
            t = time.perf_counter() - t0
            cpu = {"value": n_loc / t, "unit": "pairs/s", "cores": 1, "kind": "reference",
                   "sample": f"decode_f32_base64 of the request's {n_loc} payloads only "
                             f"({len(body) / 1e6:.1f} MB body), {t:.3f} s: an upper bound on the "
                             "reference's wire ingest rate before any scoring"}
    line = {"metric": "query-item pairs scored/sec (/score wire format, embedding_b64)",
            "value": n_loc / per_q, "unit": "pairs/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_q * 1000, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic N(0, 0.08^2) rows, base64 float32 wire payloads",
            "config": {"workload": WORKLOAD_DESC["c3_rows"] + ", items as embedding_b64 in a JSON body",
                       "body_bytes": len(body), "python_json_path_ms": py_ms},
            "e2e": {"value": n_loc / per_q, "unit": "pairs/s", "h2d_bytes_per_step": len(body),
                    "d2h_bytes_per_step": n_loc * 6 * 8,
                    "path": "ScoringEngine.score_json -> sr_wire_parse + sr_engine_score_wire"},
            "gpu_launches": None, "cpu_baseline": cpu,
            "topk_head": [(iid, round(s, 6)) for iid, s in res.topk[:3]]}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + sorted(RETRIEVAL) + ["c3_wire"],
                    default=None, help="default: c2 (configs[1]) at N=1, c5 (configs[4]) under "
                                       "torchrun with WORLD_SIZE > 1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the N=1 configs[4] sub-measurement")
    ap.add_argument("--no-serving", action="store_true",
                    help="skip the open-loop scheduler sweep (pairs/s at fixed p99)")
    args = ap.parse_args()
    if args.workload is None:
        args.workload = "c5" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "c2"
    if args.warmup < 3:
        args.warmup = 3
    if args.workload == "c3_wire":
        return 0 if args.impl == "reference" else run_wire(args)
    if args.workload in RETRIEVAL:
        if args.impl == "reference":
            return 0  # the reference arm of this contract is the ranker (configs[1])
        return run_retrieval(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
