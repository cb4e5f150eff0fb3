"""Layout reuse between calls (host/engine.cu refill_plan): a request whose
(t_q, mode, item lengths) match the plan's last layout re-uploads only its
token ids and doc ids. Results must be bit-identical to a fresh engine that
packs and uploads everything, for token and mixed requests, with changed
doc ids (the top-k tie rule reads them) and after a layout change back and
forth on one cached plan."""
import numpy as np
import pytest

import paper_2602_07309_b200 as sr
from tests.test_gpu_parity import request

pytestmark = pytest.mark.gpu


def _cfg():
    return sr.ModelConfig(n_layers=2, d_model=256, n_heads=2, d_ff=512,
                          head_specs=sr.ModelConfig.default_toy().head_specs)


def _same(a, b):
    assert np.array_equal(a.scores, b.scores)
    assert a.topk == b.topk


def _tokens(rng, lens, t_q=70):
    return (rng.integers(0, 256, t_q).astype(np.int32),
            [rng.integers(0, 256, L).astype(np.int32) for L in lens])


def test_token_requests_same_layout(cuda):
    w = sr.init_model(_cfg(), 5, "fan_in")
    warm = sr.ScoringEngine(w, device=0)
    rng = np.random.default_rng(17)
    lens = [33, 7, 96, 1, 64, 12]
    reqs = [request(*_tokens(rng, lens)) for _ in range(3)]
    # doc ids that reverse the index order: ties would resolve differently
    for i, it in enumerate(reqs[2].items):
        it.id = str(1000 - i)
    # same shape key (rows, items, tiles) -> same cached plan, other layout
    other = request(*_tokens(rng, [7, 33, 96, 1, 12, 64]))
    got = []
    for r in reqs[:2] + [other] + reqs[2:]:
        got.append(warm.score(r, k=4))
    for r, g in zip(reqs[:2] + [other] + reqs[2:], got):
        _same(g, sr.ScoringEngine(w, device=0).score(r, k=4))


def test_mixed_requests_same_layout(cuda):
    cfg = _cfg()
    w = sr.init_model(cfg, 6, "fan_in")
    warm = sr.ScoringEngine(w, device=0)
    rng = np.random.default_rng(18)
    lens = [5, 1, 9, 3]

    def mixed():
        rows = [rng.standard_normal((L, cfg.d_model)).astype(np.float32) * 0.08 for L in lens]
        return request(rng.integers(0, 256, 50).astype(np.int32), None, sr.ScoreMode.Mixed,
                       rows=rows)

    reqs = [mixed() for _ in range(3)]
    got = [warm.score(r, k=3) for r in reqs]
    for r, g in zip(reqs, got):
        _same(g, sr.ScoringEngine(w, device=0).score(r, k=3))


def test_reserve_keeps_results_and_rejects_bad_sizes(cuda):
    """sr_engine_reserve: a workspace reserved up front (the serving warm-up
    order) gives the same bits as growth on demand, for a small pass captured
    before a larger one and replayed after it."""
    w = sr.init_model(_cfg(), 5, "fan_in")
    rng = np.random.default_rng(23)
    small = request(*_tokens(rng, [40, 9, 96]))
    big = request(*_tokens(rng, [96] * 40))
    eng = sr.ScoringEngine(w, device=0)
    eng.reserve(70 + 96 * 40)
    got = [eng.score(small, k=3), eng.score(big, k=5), eng.score(small, k=3)]
    for r, k, g in zip([small, big, small], [3, 5, 3], got):
        _same(g, sr.ScoringEngine(w, device=0).score(r, k=k))
    with pytest.raises(sr.SemrankError):
        eng.reserve(0)
    with pytest.raises(sr.SemrankError):
        eng.reserve(1 << 30)
    # a reservation the device cannot hold fails cleanly; the engine recovers
    with pytest.raises(sr.SemrankError):
        eng.reserve(1 << 29)
    _same(eng.score(small, k=3), got[0])
