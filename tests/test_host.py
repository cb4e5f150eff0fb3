"""Host-side logic through the C-ABI (no GPU): exports, config/weights,
SRNKWTS1 container, FlopReport, multi-item masks, plan_batches, request
validation error categories, top-k comparator. Mirrors the reference's
test_engine.cpp / test_model.cpp cases that do not need a forward pass."""
import hashlib
import json
import os
import re

import numpy as np
import pytest

import paper_2602_07309_b200 as sr
from paper_2602_07309_b200 import _capi
from tests.refrng import Rng

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_library_exports_every_header_symbol():
    with open(os.path.join(ROOT, "include", "semrank_b200.h")) as f:
        header = re.sub(r"/\*.*?\*/", "", f.read(), flags=re.S)  # drop comments
    declared = set(re.findall(r"\b(sr_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_capi.HEADER_SYMBOLS), declared ^ set(_capi.HEADER_SYMBOLS)
    for name in declared:
        assert hasattr(_capi.lib, name), name
    assert _capi.lib.sr_abi_version() == 2


def test_status_names_mirror_error_codes():
    # error.cpp:8-27
    names = ["length_overflow", "mask_invalid", "spec_violation", "payload_invalid",
             "schema_unknown", "alignment", "divergence", "parameter", "degenerate_input",
             "undefined_metric", "state_invalid", "oversize_item", "consistency",
             "reconciliation", "io"]
    for i, n in enumerate(names, start=1):
        assert _capi.lib.sr_status_name(i).decode() == n


def test_config_validation():  # model.cpp:29-50
    cfg = sr.ModelConfig.default_toy()
    cfg.validate()
    for bad in (dict(d_model=65), dict(n_layers=0), dict(vocab_size=263), dict(no_token_id=261),
                dict(yes_token_id=400), dict(max_seq=0)):
        c = sr.ModelConfig.default_toy()
        for k, v in bad.items():
            setattr(c, k, v)
        with pytest.raises(sr.SemrankError) as e:
            c.validate()
        assert e.value.code == sr.ErrorCode.SpecViolation


def test_init_and_container_match_reference_bytes(tmp_path):
    """init_model + save_weights produce the reference's exact SRNKWTS1 bytes."""
    for name in ("toy_bench.json", "toy_ragged.json", "acceptance_c1.json"):
        g = gold(name)
        w = sr.init_model(sr.ModelConfig.default_toy(), g["seed"])
        path = str(tmp_path / "w.srnk")
        w.save(path)
        with open(path, "rb") as f:
            assert hashlib.sha256(f.read()).hexdigest() == g["weights_sha256"], name
        r = sr.load_weights(path)
        assert r.version == w.version == f"toy-{g['seed']:016x}"
        a, b = w.tensors(), r.tensors()
        assert all(np.array_equal(a[k], b[k]) for k in a)


def test_fan_in_init_matches_reference_bytes(tmp_path):
    g = gold("c2_subset.json")
    c = g["config"]
    cfg = sr.ModelConfig(n_layers=c["n_layers"], d_model=c["d_model"], n_heads=c["n_heads"],
                         d_ff=c["d_ff"], head_specs=sr.ModelConfig.default_toy().head_specs)
    w = sr.init_model(cfg, g["seed"], "fan_in")
    path = str(tmp_path / "c2.srnk")
    w.save(path)
    with open(path, "rb") as f:
        assert hashlib.sha256(f.read()).hexdigest() == g["weights_sha256"]


def test_weights_load_errors(tmp_path):
    p = tmp_path / "bad.srnk"
    p.write_bytes(b"NOTMAGIC" + b"\0" * 32)
    with pytest.raises(sr.SemrankError) as e:
        sr.load_weights(str(p))
    assert e.value.code == sr.ErrorCode.Io
    with pytest.raises(sr.SemrankError) as e:
        sr.load_weights(str(tmp_path / "missing.srnk"))
    assert e.value.code == sr.ErrorCode.Io
    w = sr.init_model(sr.ModelConfig.default_toy(), 3)
    good = tmp_path / "good.srnk"
    w.save(str(good))
    data = good.read_bytes()
    (tmp_path / "trunc.srnk").write_bytes(data[:-100])
    with pytest.raises(sr.SemrankError) as e:
        sr.load_weights(str(tmp_path / "trunc.srnk"))
    assert e.value.code == sr.ErrorCode.Io


def test_flops_closed_forms():  # test_engine.cpp:61-98
    M = sr.ScoreMode
    assert sr.flops(M.Naive, 500, 50, 100).attention_units == 30_250_000
    assert sr.flops(M.Naive, 500, 50, 100).linear_units == 55_000
    assert sr.flops(M.Ibpc, 500, 50, 100).attention_units == 5_500_000
    assert sr.flops(M.Ibpc, 500, 50, 100).linear_units == 5_500
    assert sr.flops(M.Naive, 50, 150, 50).attention_units == 2_000_000
    assert sr.flops(M.Ibpc, 50, 150, 50).attention_units == 1_877_500
    assert sr.flops(M.Ibpc, 50, 150, 50).linear_units == 7550
    assert sr.flops(M.Mixed, 40, 1, 8).attention_units == 40 * 40 + 8 * (2 * 40 + 1)
    assert sr.flops(M.Naive, 500, 50, 0).attention_units == 0
    assert sr.flops(M.Ibpc, 500, 50, 0).attention_units == 250_000
    rng = Rng(2)
    for _ in range(200):
        tq, ti, n = rng.uniform_int(1, 300), rng.uniform_int(1, 300), rng.uniform_int(1, 64)
        fn, fa = sr.flops(M.Naive, tq, ti, n), sr.flops(M.MultiItem, tq, ti, n)
        assert fa.attention_units <= fn.attention_units and fa.linear_units <= fn.linear_units
        if n >= 2:
            assert fa.attention_units < fn.attention_units
    for case in gold("host_logic.json")["flops"]:
        f = sr.flops(sr.ScoreMode(case["mode"]), case["t_q"], case["t_i"], case["n"])
        assert [f.attention_units, f.linear_units, f.t_q, f.t_i_mean, f.n_items] == case["report"]
    with pytest.raises(sr.SemrankError) as e:
        sr.flops(M.Naive, -1, 1, 1)
    assert e.value.code == sr.ErrorCode.Parameter


def test_multi_item_mask():  # test_engine.cpp:100-138
    m = sr.build_multi_item_mask(2, [2, 1])
    assert m.item_spans == [(2, 4), (4, 5)]
    attn = m.to_attention_mask()
    assert len(attn) == 3 and attn[2] == (2, 4)
    assert m.allowed_pair_count() == 13
    assert sr.build_multi_item_mask(3, [4]).allowed_pair_count() == 7 * 8 // 2
    with pytest.raises(sr.SemrankError):
        sr.build_multi_item_mask(2, [2, 0])
    rng = Rng(13)
    for _ in range(50):
        tq = rng.uniform_int(1, 12)
        lens = [rng.uniform_int(1, 9) for _ in range(rng.uniform_int(1, 6))]
        m = sr.build_multi_item_mask(tq, lens)
        expect = sum(p + 1 for p in range(tq))
        for s, e in m.item_spans:
            expect += sum(tq + (p - s + 1) for p in range(s, e))
        assert m.allowed_pair_count() == expect


def _req(prefix, lens, mode=sr.ScoreMode.MultiItem):
    r = sr.ScoreRequest(prefix_tokens=list(prefix), mode=mode)
    for i, L in enumerate(lens):
        r.items.append(sr.ScoreItem(id=f"i{i}", tokens=[2] * L))
    return r


def test_plan_batches():  # test_engine.cpp:273-342 + reference outputs
    plan = sr.plan_batches([_req([1] * 10, [5, 5, 5])], 1000)
    assert len(plan) == 1 and plan[0].token_count == 25
    plan = sr.plan_batches([_req([1] * 10, [5, 5]), _req([1] * 8, [4]), _req([1] * 6, [3, 3, 3])],
                           100)
    assert len(plan) == 1 and plan[0].token_count == 47 and len(plan[0].entries) == 3
    with pytest.raises(sr.SemrankError) as e:
        sr.plan_batches([_req([1] * 10, [100])], 50)
    assert e.value.code == sr.ErrorCode.OversizeItem
    for case in gold("host_logic.json")["plan_batches"]:
        reqs = [_req([1] * p, l) for p, l in zip(case["prefix"], case["item_lens"])]
        got = sr.plan_batches(reqs, case["budget"])
        quads = [[b, e.request_index, e.item_begin, e.item_end]
                 for b, bt in enumerate(got) for e in bt.entries]
        assert quads == case["entries"]
        assert [b.token_count for b in got] == case["batch_tokens"]


def test_request_report_matches_reference_flops():
    """FlopReport + kv per mode, including multi-item chunk re-payment."""
    g = gold("toy_bench.json")
    cfg = sr.ModelConfig.default_toy()
    for mode, name in ((0, "naive"), (1, "ibpc"), (2, "multi_item")):
        r = sr.ScoreRequest(prefix_tokens=g["prefix"], mode=sr.ScoreMode(mode),
                            items=[sr.ScoreItem(id=str(i), tokens=t) for i, t in enumerate(g["items"])])
        f, kv = sr.request_report(cfg, r)
        want = g["modes"][name]
        assert [f.attention_units, f.linear_units, f.t_q, f.t_i_mean, f.n_items] == want["flops"]
        assert kv == want["kv_incremental_per_item"]
    # chunked multi-item (engine.cpp:328-377): max_seq 64 forces several chunks
    small = sr.ModelConfig.default_toy()
    small.max_seq = 64
    r = _req([5] * 10, [8, 7, 8, 6, 8, 5, 8, 8, 4, 8, 8, 2])
    f, _ = sr.request_report(small, r)
    assert f.attention_units > sr.flops(sr.ScoreMode.MultiItem, 10, 0, 0).attention_units
    naive = _req([5] * 10, [8, 7, 8, 6, 8, 5, 8, 8, 4, 8, 8, 2], sr.ScoreMode.Naive)
    assert f.attention_units < sr.request_report(small, naive)[0].attention_units


def test_request_validation_error_categories():
    cfg = sr.ModelConfig.default_toy()
    E = sr.ErrorCode
    cases = [
        (sr.ScoreRequest(prefix_tokens=[1, 2]), E.SpecViolation),              # no items
        (_req([1, 2], [3, 0]), E.SpecViolation),                                # empty item
        (sr.ScoreRequest(prefix_tokens=[1, 300], items=[sr.ScoreItem(tokens=[1])]),
         E.SpecViolation),                                                      # OOV token
        (sr.ScoreRequest(prefix_tokens=[1] * 4000, items=[sr.ScoreItem(tokens=[1] * 200)]),
         E.LengthOverflow),                                                     # > max_seq
        (sr.ScoreRequest(prefix_tokens=[1] * 5000, items=[sr.ScoreItem(tokens=[1])]),
         E.LengthOverflow),
    ]
    for req, code in cases:
        with pytest.raises(sr.SemrankError) as e:
            sr.request_report(cfg, req)
        assert e.value.code == code, (req, e.value)
    bad = sr.ScoreRequest(prefix_tokens=[1], mode=sr.ScoreMode.Mixed,
                          items=[sr.ScoreItem(embedding=np.zeros(63, np.float32), n_emb_tokens=1)])
    with pytest.raises(sr.SemrankError) as e:
        sr.request_report(cfg, bad)
    assert e.value.code == E.PayloadInvalid


def test_topk_host_comparator():  # semrank_main.cpp:393-398, retrieval.cpp:99-102
    rng = np.random.default_rng(0)
    scores = np.round(rng.random(500) * 10) / 10
    ids = rng.permutation(5000)[:500].astype(np.int64)
    oi, os_, ox = sr.topk_host(scores, ids, 37)
    order = sorted(range(500), key=lambda i: (-scores[i], ids[i]))[:37]
    assert list(oi) == [int(ids[i]) for i in order] and list(ox) == order
    # duplicate ids keep input order (stable_sort)
    oi, _, ox = sr.topk_host(np.ones(5), np.zeros(5, np.int64), 5)
    assert list(ox) == [0, 1, 2, 3, 4]


def test_engine_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    w = sr.init_model(sr.ModelConfig.default_toy(), 1)
    with pytest.raises(sr.SemrankError) as e:
        sr.ScoringEngine(w)
    assert e.value.code == sr.ErrorCode.Cuda


# ------------------------------------------------------- native /score parser
def _wire(body, max_seq=4096):
    import ctypes as C
    from paper_2602_07309_b200._capi import lib
    raw = body.encode() if isinstance(body, str) else body
    h = C.c_void_p()
    st = lib.sr_wire_parse(raw, len(raw), max_seq, C.byref(h))
    if st != 0:
        return st, lib.sr_last_error().decode(), None
    n, mode, tq = C.c_int32(), C.c_int32(), C.c_int32()
    lib.sr_wire_info(h, C.byref(n), C.byref(mode), C.byref(tq))
    info = (n.value, mode.value, tq.value, lib.sr_wire_request_id(h).decode(),
            [lib.sr_wire_item_id(h, i).decode() for i in range(n.value)])
    lib.sr_wire_destroy(h)
    return 0, "", info


def test_native_wire_parser_follows_parse_score_request_json():
    """service.cpp:326-372: fields, defaults, precedence and error messages."""
    import json
    import paper_2602_07309_b200 as sr
    body = json.dumps({"request_id": "réq", "prefix_text": "hi \"there\"", "mode": "multi-item",
                       "extra": {"nested": [1, {"x": None}]},
                       "items": [{"id": "7", "text": "a\\nb"}, {"id": "9", "tokens": [1, 2]},
                                 {"tokens": [3], "text": "ignored", "id": "11"}]})
    st, msg, info = _wire(body)
    assert st == 0, msg
    n, mode, tq, rid, ids = info
    assert (n, mode, tq, rid, ids) == (3, int(sr.ScoreMode.MultiItem), len(b'hi "there"'), "réq",
                                       ["7", "9", "11"])
    # default mode is ibpc (service.cpp:343)
    assert _wire('{"prefix_tokens":[1],"items":[{"tokens":[2]}]}')[2][1] == int(sr.ScoreMode.Ibpc)
    P = int(sr.ErrorCode.PayloadInvalid)
    cases = [("{not json", P, "request body is not JSON"),
             ('{"items":[{"tokens":[1]}]}', P, "request needs prefix_text or prefix_tokens"),
             ('{"prefix_tokens":[1],"items":[]}', P, "request needs a non-empty items[]"),
             ('{"prefix_tokens":[1],"items":{}}', P, "request needs a non-empty items[]"),
             ('{"prefix_tokens":[1],"items":[{"id":"q"}]}', P,
              "item needs text, tokens, or embedding_b64: q"),
             ('{"prefix_tokens":[1],"mode":"bogus","items":[{"tokens":[1]}]}',
              int(sr.ErrorCode.Parameter), "unknown scoring mode: bogus"),
             ('{"prefix_text":"abcdef","items":[{"tokens":[1]}]}', int(sr.ErrorCode.LengthOverflow),
              "exceeds max_seq 4")]
    for body, code, text in cases:
        st, msg, _ = _wire(body, max_seq=4)
        assert st == code and text in msg, (body, st, msg)


def _grouped(filters):
    out = {}
    for a, v in filters:
        out.setdefault(a, []).append(v)
    return out


def test_canonical_query_and_signature_match_reference_golden():
    """midtier.cpp:14-53 (test_midtier.cpp:18-25 plus whitespace / case /
    non-ASCII / multi-attribute cases), golden from oracle/_ref."""
    g = gold("score_cache.json")
    for c in g["queries"]:
        f = _grouped(c["filters"])
        assert sr.canonical_query(c["text"], f) == c["canonical"], c
        assert sr.query_signature(c["text"], f) == int(c["fnv1a64"]), c
        assert sr.fnv1a64(c["canonical"]) == int(c["fnv1a64"])
    assert sr.fnv1a64("") == 1469598103934665603  # midtier.cpp:47's basis


def test_score_cache_lru_traces_match_reference_golden():
    """ScoreCache (midtier.cpp:64-100): hits, misses, recency, eviction,
    idempotent and conflicting puts, replayed from the reference's traces."""
    g = gold("score_cache.json")
    for t in g["traces"]:
        cache = sr.ScoreCache(t["capacity"], task_names=["relevance"])
        for (op, who, sig, ent, ver, val), (want, want_val, want_size) in zip(t["ops"], t["out"]):
            key = sr.CacheKey(who, int(sig), int(ent), ver)
            if op == 0:
                got = cache.get(key)
                assert (got is not None) == bool(want)
                if got is not None:
                    assert got["relevance"] == want_val
            else:
                try:
                    cache.put(key, {"relevance": val})
                    st = 0
                except sr.SemrankError as e:
                    st = int(e.code)
                    assert "conflicting scores for one cache key" in str(e)
                assert st == want
            assert cache.size() == want_size
        assert cache.capacity() == t["capacity"]
    with pytest.raises(sr.SemrankError) as ei:
        sr.ScoreCache(0)
    assert int(ei.value.code) == g["zero_capacity"]["status"]
    assert g["zero_capacity"]["message"] in str(ei.value)


def test_score_cache_concurrent_readers_and_writers():
    """test_midtier.cpp / test_service.cpp:393-410: one mutex, no lost entries."""
    import threading
    cache = sr.ScoreCache(64, task_names=["relevance"])

    def work(t):
        for i in range(200):
            key = sr.CacheKey("s", t, i % 32, "v")
            cache.put(key, {"relevance": float(i % 32)})
            got = cache.get(key)
            assert got is None or got["relevance"] == float(i % 32)

    ths = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert cache.size() <= 64
