"""Randomised parity on the tcgen05 path: a small model whose shapes take the
production kernels (d 256 = 2 heads of 128: CTA-pair GEMMs with every fused
epilogue, the tcgen05 attention, the row kernels) scored on random requests
— prefix lengths, item counts and lengths, token and mixed modes — against
the C oracle on bf16-rounded weights, one request at a time and several
packed into one device pass (plan_batches generalised, engine.cpp:278-326).

Tolerance as tests/test_gpu_parity.py (TOL = 6e-3 on probabilities); top-k
equals the oracle order outside ties (2 x the measured deviation)."""
import numpy as np
import pytest

import paper_2602_07309_b200 as sr
from oracle import oracle as O
from tests.test_gpu_parity import TOL, assert_topk_outside_ties, request

pytestmark = pytest.mark.gpu


def _cfg():
    return sr.ModelConfig(n_layers=2, d_model=256, n_heads=2, d_ff=512,
                          head_specs=sr.ModelConfig.default_toy().head_specs)


def _random_request(rng, d, mixed):
    t_q = int(rng.integers(1, 300))
    n = int(rng.integers(1, 40))
    prefix = rng.integers(0, 256, t_q).astype(np.int32)
    if mixed:
        rows = [rng.standard_normal((int(rng.integers(1, 24)), d)).astype(np.float32) * 0.08
                for _ in range(n)]
        return prefix, None, rows
    items = [rng.integers(0, 256, int(rng.integers(1, 200))).astype(np.int32) for _ in range(n)]
    return prefix, items, None


def test_random_requests_single_and_batched(cuda):
    cfg = _cfg()
    eng = sr.ScoringEngine(sr.init_model(cfg, 77, "fan_in"), device=0)
    ow = O.OracleWeights.init(cfg, 77, 1)
    ow.round_bf16()
    rng = np.random.default_rng(4242)
    cases, reqs = [], []
    worst = 0.0
    for trial in range(24):
        mixed = trial % 3 == 2
        prefix, items, rows = _random_request(rng, cfg.d_model, mixed)
        mode = sr.ScoreMode.Mixed if mixed else sr.ScoreMode.MultiItem
        req = request(prefix, items, mode, rows=rows)
        ref = ow.score(prefix, items=items, rows=rows)
        res = eng.score(req, k=5)
        dev = float(np.abs(res.scores - ref).max())
        worst = max(worst, dev)
        assert dev <= TOL, f"trial {trial}: max |dp| {dev:.2e}"
        assert_topk_outside_ties([int(i) for i, _ in res.topk], ref[:, 0], min(5, len(ref)),
                                 res.scores[:, 0])
        cases.append(ref)
        reqs.append(req)
    # the same requests, four at a time in one packed pass (mixed modes together)
    for lo in range(0, len(reqs), 4):
        got = eng.score_batch(reqs[lo:lo + 4], k=5)
        for r, ref in zip(got, cases[lo:lo + 4]):
            assert float(np.abs(r.scores - ref).max()) <= TOL
    print(f"24 random requests: max |dp| vs oracle {worst:.2e}")
