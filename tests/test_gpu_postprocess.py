"""Service post-processing on the device: calibrated
relevance + score blend as the page's ranking key (service.cpp:242-277),
bit-identical to the C restatement (pinned to the reference's calibrate by
tests/golden/calibration.json) applied to the same raw scores."""
import json
import os

import numpy as np
import pytest

import paper_2602_07309_b200 as sr
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "calibration.json")


def head():
    with open(GOLD) as f:
        g = json.load(f)
    F = lambda k: [float(x) for x in g[k]]
    return sr.CalibrationHead([sr.CalibrationBlock(a, b, c) for a, b, c in
                               zip(F("lo"), F("hi"), F("value"))])


def toy_request(n=64, seed=1):
    prefix, items = O.bench_tokens(seed, 500, 50, n)
    req = sr.ScoreRequest(request_id="pp", prefix_tokens=prefix, mode=sr.ScoreMode.MultiItem,
                          items=[sr.ScoreItem(id=str(1000 - i), tokens=t) for i, t in enumerate(items)])
    return req


def expected_order(final, ids, k):
    return sorted(range(len(final)), key=lambda i: (-final[i], ids[i]))[:k]


@pytest.mark.parametrize("blend", [None, {"relevance": 0.7, "click": 0.2, "apply": 0.1},
                                   {"dismiss": -1.0, "relevance": 2.0}])
def test_calibrated_blend_ranking_matches_oracle(cuda, blend):
    eng = sr.ScoringEngine(sr.init_model(sr.ModelConfig.default_toy(), 1), device=0)
    h = head()
    eng.set_postprocess(h, blend)
    req = toy_request()
    res = eng.score(req, k=10)
    names = ["relevance"] + list(eng.task_names[1:])
    bt = [names.index(t) for t in sorted(blend)] if blend else []
    bw = [blend[t] for t in sorted(blend)] if blend else []
    want = O.oracle_final_scores(res.scores, [b.lo for b in h.blocks], [b.hi for b in h.blocks],
                                 [b.value for b in h.blocks], bt, bw)
    assert np.array_equal(res.final_scores, want)
    ids = [int(it.id) for it in req.items]
    order = expected_order(want, ids, 10)
    assert [str(ids[i]) for i in order] == [iid for iid, _ in res.topk]
    assert [s for _, s in res.topk] == [want[i] for i in order]
    # off again: top-k by raw relevance
    eng.set_postprocess(None, None)
    res2 = eng.score(req, k=10)
    rel = res2.scores[:, 0]
    assert [iid for iid, _ in res2.topk] == [str(ids[i]) for i in expected_order(rel, ids, 10)]


def test_unknown_blend_task_is_an_alignment_error(cuda):
    eng = sr.ScoringEngine(sr.init_model(sr.ModelConfig.default_toy(), 1), device=0)
    with pytest.raises(sr.SemrankError) as e:
        eng.set_postprocess(head(), {"relevance": 1.0, "nope": 0.5})
    assert e.value.code == sr.ErrorCode.Alignment


def test_blend_without_fitted_head_is_state_invalid(cuda):
    # calibration.cpp:65-68: calibrate() on an unfitted head throws StateInvalid;
    # the C-ABI refuses the same configuration
    eng = sr.ScoringEngine(sr.init_model(sr.ModelConfig.default_toy(), 1), device=0)
    with pytest.raises(sr.SemrankError) as e:
        eng.set_postprocess(None, {"relevance": 1.0})
    assert e.value.code == sr.ErrorCode.StateInvalid
    import ctypes as C
    from paper_2602_07309_b200._capi import lib
    t = (C.c_int32 * 1)(0)
    w = (C.c_double * 1)(1.0)
    z = (C.c_double * 1)(0.0)
    assert lib.sr_engine_set_postprocess(eng._h, z, z, z, 0, t, w, 1) == int(sr.ErrorCode.StateInvalid)
