"""build_prompt (prompt.cpp:14-38) and score_result_to_json
(service.cpp:380-391) through the library, against golden outputs of the
reference itself (tests/golden/text_api.json, oracle/gen_golden.py text_api:
build_prompt compiled from the reference sources; the response bodies
serialised by the reference's nlohmann::json)."""
import base64
import json
import os

import numpy as np
import pytest

import paper_2602_07309_b200 as sr

GOLD = os.path.join(os.path.dirname(__file__), "golden", "text_api.json")


def _raw(b64):
    return base64.b64decode(b64) if b64 else b""


@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


def test_build_prompt_matches_reference(gold):
    for case in gold["prompts"]:
        args = (_raw(case["system"]), _raw(case["query"]), _raw(case["document"]), case["max_seq"])
        if case["status"] == 0:
            parts = sr.build_prompt(*args)
            assert parts.prefix_tokens == case["prefix"] and parts.item_tokens == case["item"]
            assert bytes(parts.item_tokens).endswith(sr.kPromptSuffix.encode())
        else:
            with pytest.raises(sr.SemrankError) as e:
                sr.build_prompt(*args)
            assert e.value.code == case["status"]  # both 1 + semrank::ErrorCode
            assert case["message"] in str(e.value)


def _result(body):
    names = body["names"]
    sc = np.array([[float(v) for v in row] for row in body["scores"]], np.float64)
    items = [sr.ItemScores(_raw(i).decode("utf-8"), {n: float(sc[j, t]) for t, n in enumerate(names)})
             for j, i in enumerate(body["ids"])]
    fl = sr.FlopReport(float(body["attention"]), float(body["linear"]), 0.0, 0.0, 0.0)
    return sr.ScoreResult(request_id=_raw(body["request_id"]).decode("utf-8"), items=items, flops=fl)


def test_score_result_to_json_bytes_match_reference(gold):
    for body in gold["bodies"]:
        assert sr.score_result_to_json(_result(body)) == body["json"]


def test_score_result_to_json_round_trips_doubles(gold):
    body = gold["bodies"][-1]
    parsed = json.loads(sr.score_result_to_json(_result(body)))
    got = [e["tasks"]["relevance"] for e in parsed["scores"]]
    want = [float(r[0]) for r in body["scores"]]
    assert all(a == b and np.signbit(a) == np.signbit(b) for a, b in zip(got, want))


def test_score_result_to_json_rejects_invalid_utf8():
    res = sr.ScoreResult(request_id="r", items=[sr.ItemScores("ok", {"relevance": 0.5})])
    res.items[0].item_id = b"\xff".decode("latin-1")  # encodes to valid UTF-8 (U+00FF)
    assert "ÿ" in sr.score_result_to_json(res)
    import ctypes as C
    from paper_2602_07309_b200 import _capi
    ids = (C.c_char_p * 1)(b"\xff")
    names = (C.c_char_p * 1)(b"relevance")
    sc = np.zeros(1)
    n = C.c_int64(0)
    st = _capi.lib.sr_score_result_to_json(b"r", 1, ids, 1, names,
                                           sc.ctypes.data_as(C.POINTER(C.c_double)),
                                           C.byref(_capi.FlopReportC()), None, 0, C.byref(n))
    assert st == sr.ErrorCode.PayloadInvalid
