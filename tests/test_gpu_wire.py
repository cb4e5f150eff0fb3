"""/score wire ingest on the device: embedding_b64 items
(service.cpp:361-370) decoded in HBM (kernels/wire.cu) with the reference's
decode_f32_base64 semantics (base64.cpp:60-108, pinned by
tests/golden/wire_b64.json from oracle/_ref)."""
import base64
import json
import os

import numpy as np
import pytest

import paper_2602_07309_b200 as sr

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "wire_b64.json")


def toy_engine():
    return sr.ScoringEngine(sr.init_model(sr.ModelConfig.default_toy(), 1), device=0)


def body(prefix, payloads, ids=None):
    items = [{"id": str(ids[i] if ids is not None else i), "embedding_b64": p}
             for i, p in enumerate(payloads)]
    return json.dumps({"request_id": "w", "prefix_tokens": list(map(int, prefix)),
                       "mode": "mixed", "items": items})


def test_b64_items_score_bit_identical_to_float_rows(cuda):
    """Decoding on the device yields the same rows, so the same scores."""
    eng = toy_engine()
    d = eng.config.d_model
    rng = np.random.default_rng(4)
    prefix = rng.integers(0, 256, 120)
    rows = [rng.standard_normal((int(rng.integers(1, 4)), d)).astype(np.float32) * np.float32(0.08)
            for _ in range(37)]  # 1-3 rows each: every base64 padding length occurs
    req_f = sr.ScoreRequest(prefix_tokens=list(prefix), mode=sr.ScoreMode.Mixed,
                            items=[sr.ScoreItem(id=str(i), embedding=r, n_emb_tokens=len(r))
                                   for i, r in enumerate(rows)])
    want = eng.score(req_f, k=5)
    req_w = sr.parse_score_request_json(
        body(prefix, [base64.b64encode(r.tobytes()).decode() for r in rows]), d)
    got = eng.score(req_w, k=5)
    assert np.array_equal(got.scores, want.scores)
    assert got.topk == want.topk


def test_c3_shaped_wire_request(cuda):
    cfg = sr.ModelConfig(n_layers=2, d_model=1024, n_heads=8, d_ff=1536,
                         head_specs=sr.ModelConfig.default_toy().head_specs)
    eng = sr.ScoringEngine(sr.init_model(cfg, 2026, "fan_in"))
    rng = np.random.default_rng(5)
    rows = rng.standard_normal((256, 8, 1024)).astype(np.float32) * np.float32(0.08)
    prefix = rng.integers(0, 256, 256)
    want = eng.score(sr.ScoreRequest(prefix_tokens=list(prefix), mode=sr.ScoreMode.Mixed,
                                     items=[sr.ScoreItem(id=str(i), embedding=rows[i],
                                                         n_emb_tokens=8) for i in range(256)]), k=10)
    req = sr.parse_score_request_json(
        body(prefix, [base64.b64encode(r.tobytes()).decode() for r in rows]), 1024)
    got = eng.score(req, k=10)
    assert np.array_equal(got.scores, want.scores)


def _expect_payload_error(eng, prefix, payloads, message):
    req = sr.parse_score_request_json(body(prefix, payloads), eng.config.d_model)
    with pytest.raises(sr.SemrankError) as e:
        eng.score(req, k=3)
    assert e.value.code == sr.ErrorCode.PayloadInvalid
    assert message in str(e.value), str(e.value)


def test_reference_decode_errors(cuda):
    """Every malformed payload of the golden set, as the last item of an
    otherwise valid request: the engine raises the reference's error."""
    eng = toy_engine()
    d = eng.config.d_model
    good = base64.b64encode(np.zeros(d, np.float32).tobytes()).decode()
    with open(GOLD) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        if c["status"] == 0:
            continue
        _expect_payload_error(eng, [1, 2, 3], [good, c["text"]], c["message"])


def test_first_failing_item_wins(cuda):
    """The reference decodes items in order: a bad character in item 0 is
    reported before a bad length in item 1, and a bad length in item 0
    before a bad character in item 1."""
    eng = toy_engine()
    d = eng.config.d_model
    good = base64.b64encode(np.ones(d, np.float32).tobytes()).decode()
    bad_char = good[:10] + "!" + good[11:]
    _expect_payload_error(eng, [7], [bad_char, good[:-1]], "invalid base64 character")
    _expect_payload_error(eng, [7], [good[:-1], bad_char], "base64 length must be mod 4")
    # whole floats but not [n x d]
    _expect_payload_error(eng, [7], [good, base64.b64encode(np.ones(d + 1, np.float32).tobytes())
                                     .decode()], f"is not [n x {d}]")
    # an error in a later item still fails the whole request, after device decode
    _expect_payload_error(eng, [7], [good, good[:-8] + "AAA=AAAA"], "misplaced base64 padding")


def test_native_wire_path_matches_python_parse(cuda):
    """ScoringEngine.score_json (native one-pass parser, payload spans of the
    body decoded in HBM) == parse_score_request_json + score, bit for bit;
    JSON escapes inside a payload ("\\/") and token / text items included."""
    eng = toy_engine()
    d = eng.config.d_model
    rng = np.random.default_rng(8)
    prefix = rng.integers(0, 256, 64)
    rows = [rng.standard_normal((int(rng.integers(1, 4)), d)).astype(np.float32) * np.float32(0.08)
            for _ in range(23)]
    pays = [base64.b64encode(r.tobytes()).decode() for r in rows]
    b = body(prefix, pays, ids=list(range(100, 123)))
    # escape every '/' of one payload the way some JSON encoders do
    k = next(i for i, p in enumerate(pays) if "/" in p)
    b = b.replace(pays[k], pays[k].replace("/", "\\/"))
    got = eng.score_json(b, k=5)
    want = eng.score(sr.parse_score_request_json(b, d), k=5)
    assert np.array_equal(got.scores, want.scores) and got.topk == want.topk
    assert [it.item_id for it in got.items] == [str(i) for i in range(100, 123)]
    assert got.request_id == want.request_id and got.mode == want.mode
    assert got.items[3].tasks == want.items[3].tasks
    toks = json.dumps({"request_id": "t", "prefix_text": "query: shoes", "mode": "multi_item",
                       "items": [{"id": str(i), "text": f"item {i} text"} for i in range(40)]})
    got = eng.score_json(toks, k=7)
    want = eng.score(sr.parse_score_request_json(toks, d), k=7)
    assert np.array_equal(got.scores, want.scores) and got.topk == want.topk
    with pytest.raises(sr.SemrankError) as e:
        eng.score_json(body(prefix, [pays[0], pays[1][:-1]]), k=2)
    assert "base64 length must be mod 4" in str(e.value)
