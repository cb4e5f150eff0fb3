"""End-to-end engine checks against the PyTorch fp32 restatement (tests/torch_ref.py).

Oracle parity (the reference's own CPU code) lives in test_gpu_parity.py;
these cases catch gross kernel/wiring errors with an independent reference.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _request(rng, t_q, lens, mode=None):
    import paper_2602_07309_b200 as sr
    req = sr.ScoreRequest(request_id="r", prefix_tokens=[int(x) for x in rng.integers(0, 256, t_q)])
    for i, L in enumerate(lens):
        req.items.append(sr.ScoreItem(id=str(i), tokens=[int(x) for x in rng.integers(0, 256, L)]))
    req.mode = mode if mode is not None else sr.ScoreMode.MultiItem
    return req


@pytest.mark.parametrize("scheme,t_q,lens", [
    ("reference", 50, [150, 7, 33, 1]),
    ("reference", 500, [50] * 8),
    ("fan_in", 64, [20, 64, 65]),
])
def test_toy_engine_matches_torch_fp32(cuda, scheme, t_q, lens):
    import paper_2602_07309_b200 as sr
    from tests.torch_ref import forward_items
    cfg = sr.ModelConfig.default_toy()
    w = sr.init_model(cfg, 1, scheme)
    eng = sr.ScoringEngine(w)
    rng = np.random.default_rng(t_q)
    req = _request(rng, t_q, lens)
    res = eng.score(req, k=3)
    ref = forward_items(w, cfg, req.prefix_tokens, [it.tokens for it in req.items], cuda)
    for got, want in zip(res.items, ref):
        for task, p in want.items():
            assert abs(got.tasks[task] - p) < 2e-2, (task, got.tasks[task], p)
    rel = [it.tasks["relevance"] for it in res.items]
    best = sorted(range(len(rel)), key=lambda i: (-rel[i], i))[:3]
    assert [int(i) for i, _ in res.topk] == best


def test_c2_shape_engine_matches_torch_fp32(cuda):
    import paper_2602_07309_b200 as sr
    from tests.torch_ref import forward_items
    cfg = sr.ModelConfig(n_layers=4, d_model=1024, n_heads=8, d_ff=1536,
                         head_specs=sr.ModelConfig.default_toy().head_specs)
    w = sr.init_model(cfg, 2026, "fan_in")
    eng = sr.ScoringEngine(w)
    rng = np.random.default_rng(7)
    req = _request(rng, 256, [96] * 5)
    res = eng.score(req, k=5)
    ref = forward_items(w, cfg, req.prefix_tokens, [it.tokens for it in req.items], cuda)
    dev = max(abs(g.tasks[t] - p) for g, r in zip(res.items, ref) for t, p in r.items())
    assert dev < 1e-2, dev


def test_modes_agree_and_mixed_substitute_embedding(cuda):
    import paper_2602_07309_b200 as sr
    cfg = sr.ModelConfig.default_toy()
    w = sr.init_model(cfg, 1)
    eng = sr.ScoringEngine(w)
    rng = np.random.default_rng(3)
    req = _request(rng, 40, [12, 5, 9])
    outs = []
    for m in (sr.ScoreMode.Naive, sr.ScoreMode.Ibpc, sr.ScoreMode.MultiItem):
        req.mode = m
        outs.append(eng.score(req).scores)
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    tok = w.tensors()["tok_emb"].reshape(cfg.vocab_size, cfg.d_model)
    mixed = sr.ScoreRequest(prefix_tokens=req.prefix_tokens, mode=sr.ScoreMode.Mixed)
    for it in req.items:
        mixed.items.append(sr.ScoreItem(id=it.id, embedding=tok[list(it.tokens)].copy(),
                                        n_emb_tokens=len(it.tokens)))
    got = eng.score(mixed).scores
    assert np.array_equal(got, outs[0])
