"""Serving scheduler on the device: requests submitted concurrently are packed
into multi-request passes and every request's scores and top-k are bit-identical
to its own sr_engine_score call (requests start on attention-tile boundaries in
a packed pass, so the composition of a pass never changes a request's bits)."""
import threading

import numpy as np
import pytest

import paper_2602_07309_b200 as sr
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _requests(n, seed=3):
    rng = np.random.default_rng(seed)
    out = []
    for q in range(n):
        t_q = int(rng.integers(20, 120))
        r = sr.ScoreRequest(request_id=f"q{q}", prefix_tokens=rng.integers(0, 256, t_q).tolist(),
                            mode=sr.ScoreMode.MultiItem)
        for i in range(int(rng.integers(1, 40))):
            r.items.append(sr.ScoreItem(id=f"{q}:{i}",
                                        tokens=rng.integers(0, 256, int(rng.integers(1, 60))).tolist()))
        out.append(r)
    return out


def test_scheduler_passes_equal_single_calls(cuda):
    eng = sr.ScoringEngine(sr.init_model(sr.ModelConfig.default_toy(), 1), device=0)
    reqs = _requests(48)
    solo = [eng.score(r, k=5) for r in reqs]
    got = {}
    with sr.Scheduler(eng, k=5, max_queries=8, max_wait_us=2000) as s:
        def client(c):
            for r in reqs[c::4]:
                got[r.request_id] = s.wait(s.submit(r))
        th = [threading.Thread(target=client, args=(c,)) for c in range(4)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        st = s.stats()
    assert st["completed"] == 48 and st["failed"] == 0
    assert st["mean_batch"] > 1.0  # concurrent callers shared passes
    for r, a in zip(reqs, solo):
        b, lat, nb = got[r.request_id]
        assert np.array_equal(a.scores, b.scores), r.request_id
        assert a.topk == b.topk
        assert lat > 0 and nb >= 1
        assert b.flops.n_items == len(r.items)


def test_scheduler_c2_scale_against_oracle_and_budget(cuda):
    """Two C2-shape queries through the scheduler under a latency budget: both
    in range of the bf16-weight oracle on a sample of items, and the learned
    per-row pass time is positive."""
    cfg = sr.ModelConfig(n_layers=2, d_model=1024, n_heads=8, d_ff=1536,
                         head_specs=sr.ModelConfig.default_toy().head_specs)
    w = sr.init_model(cfg, 2026, "fan_in")
    eng = sr.ScoringEngine(w, device=0)
    rng = np.random.default_rng(11)
    reqs = []
    for q in range(2):
        r = sr.ScoreRequest(request_id=f"c{q}", prefix_tokens=rng.integers(0, 256, 256).tolist(),
                            mode=sr.ScoreMode.MultiItem)
        for i in range(64):
            r.items.append(sr.ScoreItem(id=str(i), tokens=rng.integers(0, 256, 96).tolist()))
        reqs.append(r)
    with sr.Scheduler(eng, k=10, max_queries=4, budget_ms=200.0) as s:
        ts = [s.submit(r) for r in reqs]
        outs = [s.wait(t) for t in ts]
        assert s.stats()["ms_per_row"] > 0
    ow = O.OracleWeights.init(cfg, 2026, 1)  # fan-in, byte-identical to init_model
    ow.round_bf16()
    for r, (res, _, _) in zip(reqs, outs):
        ref = ow.score(r.prefix_tokens, [it.tokens for it in r.items[:8]])
        assert float(np.abs(res.scores[:8] - ref).max()) < 5e-3
        assert np.array_equal(res.scores, eng.score(r, k=10).scores)
