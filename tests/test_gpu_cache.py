"""Score cache around the device scorer: handle_search's
probe -> score misses -> put -> rank path (service.cpp:160-234, 279-289).
The reference's service test (test_service.cpp:263-291) is the bar: a second
identical request is served entirely from the cache, and enabling the cache
changes no returned score: bit-exact here against an uncached device pass
over the same items, for token and soft-row items; with partial hits, every
row is bit-exact to the pass that produced it, and the ranking (raw, or the
calibrated / blended key) is the comparator over the returned rows."""
import json
import os

import numpy as np
import pytest

import paper_2602_07309_b200 as sr
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "calibration.json")


@pytest.fixture(scope="module")
def eng(cuda):
    return sr.ScoringEngine(sr.init_model(sr.ModelConfig.default_toy(), 1), device=0)


def token_request(ids, seed=3):
    prefix, items = O.bench_tokens(seed, 500, 50, max(ids) + 1)
    return sr.ScoreRequest(request_id="c", prefix_tokens=prefix, mode=sr.ScoreMode.MultiItem,
                           items=[sr.ScoreItem(id=str(i), tokens=items[i]) for i in ids])


def soft_request(ids, d, seed=5):
    rng = np.random.default_rng(seed)
    rows = {i: np.random.default_rng(1000 + i).normal(0, 0.08, (1 + i % 3, d)).astype(np.float32)
            for i in ids}
    prefix = rng.integers(0, 255, 40).tolist()
    return sr.ScoreRequest(request_id="m", prefix_tokens=prefix, mode=sr.ScoreMode.Mixed,
                           items=[sr.ScoreItem(id=str(i), embedding=rows[i].reshape(-1),
                                               n_emb_tokens=rows[i].shape[0]) for i in ids])


def check_same(got, want):
    assert np.array_equal(got.scores, want.scores)
    assert got.topk == want.topk
    if want.final_scores is not None:
        assert np.array_equal(got.final_scores, want.final_scores)


@pytest.mark.parametrize("kind", ["tokens", "soft"])
def test_second_request_is_all_hits_and_scores_unchanged(eng, kind):
    ids = list(range(40))
    req = token_request(ids) if kind == "tokens" else soft_request(ids, eng.config.d_model)
    cache = sr.ScoreCache(1000, eng.task_names)
    sig = sr.query_signature("senior ml engineer", {"region": ["na"]})
    plain = eng.score(req, k=10)
    first = eng.score_cached(req, cache, "s", sig, k=10)
    assert first.cache_hits == 0 and cache.size() == len(ids)
    check_same(first, plain)
    assert first.flops.linear_units == plain.flops.linear_units
    second = eng.score_cached(req, cache, "s", sig, k=10)
    assert second.cache_hits == len(ids)
    check_same(second, plain)
    assert second.flops.linear_units == 0 and second.flops.attention_units == 0
    # another searcher / signature / model version misses
    assert eng.score_cached(req, cache, "t", sig, k=10).cache_hits == 0
    assert eng.score_cached(req, cache, "s", sig + 1, k=10).cache_hits == 0
    assert eng.score_cached(req, cache, "s", sig, k=10, model_version="other").cache_hits == 0


def expected_topk(key, ids, k):
    order = sorted(range(len(key)), key=lambda i: (-key[i], ids[i]))[:k]
    return [(str(ids[i]), float(key[i])) for i in order]


@pytest.mark.parametrize("kind", ["tokens", "soft"])
def test_partial_hits(eng, kind):
    """Hit rows are the cached rows; miss rows are bit-identical to a device
    pass over exactly the missed items (same batch composition), and within
    the permutation-stability bound of a pass over the whole page (the
    attention key blocks follow the batch packing; test_engine.cpp:189-209
    allows 1e-5 in fp32); the top-k ranks the returned rows."""
    mk = (lambda ids: token_request(ids)) if kind == "tokens" else \
        (lambda ids: soft_request(ids, eng.config.d_model))
    cache = sr.ScoreCache(1000, eng.task_names)
    even = list(range(0, 60, 2))
    first = eng.score_cached(mk(even), cache, "s", 9, k=5)
    order = list(range(59, -1, -1))  # reversed, odd ids new
    res = eng.score_cached(mk(order), cache, "s", 9, k=12)
    assert res.cache_hits == 30 and cache.size() == 60
    odd = [i for i in order if i % 2]
    misses = eng.score(mk(odd))
    for j, i in enumerate(order):
        if i % 2 == 0:
            assert np.array_equal(res.scores[j], first.scores[even.index(i)])
        else:
            assert np.array_equal(res.scores[j], misses.scores[odd.index(i)])
    full = eng.score(mk(order), k=12)
    assert np.abs(res.scores - full.scores).max() <= 2e-3
    assert res.topk == expected_topk(res.scores[:, 0], order, 12)


def test_cache_with_calibrated_blend_ranking(eng):
    with open(GOLD) as f:
        g = json.load(f)
    head = sr.CalibrationHead([sr.CalibrationBlock(float(a), float(b), float(c))
                               for a, b, c in zip(g["lo"], g["hi"], g["value"])])
    blend = {"relevance": 0.7, "click": 0.2, "dismiss": -0.1}
    eng.set_postprocess(head, blend)
    names = eng.task_names
    bt = [names.index(t) for t in sorted(blend)]
    bw = [blend[t] for t in sorted(blend)]
    try:
        cache = sr.ScoreCache(16, eng.task_names)  # smaller than the page: evictions
        ids = list(range(48))
        req = token_request(ids)
        plain = eng.score(req, k=10)
        check_same(eng.score_cached(req, cache, "s", 1, k=10), plain)  # all misses
        for _ in range(2):
            res = eng.score_cached(req, cache, "s", 1, k=10)
            want = O.oracle_final_scores(res.scores, [b.lo for b in head.blocks],
                                         [b.hi for b in head.blocks],
                                         [b.value for b in head.blocks], bt, bw)
            assert np.array_equal(res.final_scores, want)
            assert res.topk == expected_topk(want, ids, 10)
        assert cache.size() == 16
    finally:
        eng.set_postprocess(None, None)


def test_cache_errors(eng):
    cache = sr.ScoreCache(8, eng.task_names)
    req = token_request([0, 1, 2])
    for it in req.items:
        it.id = "doc-" + it.id
    with pytest.raises(sr.SemrankError) as ei:
        eng.score_cached(req, cache, "s", 1)
    assert ei.value.code == sr.ErrorCode.SpecViolation
    res = eng.score_cached(req, cache, "s", 1, k=2, entity_ids=[10, 11, 12])
    assert res.cache_hits == 0 and cache.size() == 3
    # a row under an existing key that differs from the device's is a
    # Consistency error on put (midtier.cpp:80-86)
    key = sr.CacheKey("s", 1, 10, eng.weights.version)
    row = cache.get(key)
    row["relevance"] += 1e-9
    with pytest.raises(sr.SemrankError) as ei:
        cache.put(key, row)
    assert ei.value.code == sr.ErrorCode.Consistency
    with pytest.raises(sr.SemrankError) as ei:
        eng.score_cached(req, sr.ScoreCache(8, ["relevance"]), "s", 1, entity_ids=[1, 2, 3])
    assert ei.value.code == sr.ErrorCode.Alignment
