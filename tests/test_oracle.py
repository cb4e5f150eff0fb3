"""Pins the CPU oracle (oracle/semrank_oracle.c) to the reference.

Golden vectors in tests/golden/ were produced by the reference's own code
(oracle/gen_golden.py running oracle/_ref = /root/reference/proj sources
compiled in place). The C restatement must reproduce them bit for bit.
When oracle/_ref is present (this container), extra fuzz cases compare the
port and the reference directly.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.refrng import Rng, random_request

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


class Cfg:
    def __init__(self, c):
        self.n_layers, self.d_model, self.n_heads = c["n_layers"], c["d_model"], c["n_heads"]
        self.d_ff, self.vocab_size, self.max_seq = c["d_ff"], c["vocab_size"], c["max_seq"]
        self.yes_token_id, self.no_token_id = 261, 262

        class H:
            def __init__(self, n):
                self.name, self.arity = n, 1
        self.head_specs = [H(n) for n in c["heads"]]


def port_weights(g, scheme=0, tmp=None):
    cfg = Cfg(g["config"])
    w = O.OracleWeights.init(cfg, g["seed"], scheme)
    if tmp is not None:
        path = os.path.join(tmp, "w.srnk")
        w.save(path)
        with open(path, "rb") as f:
            assert hashlib.sha256(f.read()).hexdigest() == g["weights_sha256"], \
                "port init/container differs from the reference's init_model + save_weights"
    return w


def test_rng_stream_matches_reference():
    g = gold("rng_stream.json")
    r = Rng(g["seed"])
    assert [r.uniform_int(g["lo"], g["hi"]) for _ in g["values"]] == g["values"]
    assert list(O.uniform_ints(g["seed"], g["lo"], g["hi"], len(g["values"]))) == g["values"]


def test_toy_bench_bit_exact(tmp_path):
    g = gold("toy_bench.json")
    w = port_weights(g, 0, str(tmp_path))
    p, items = O.bench_tokens(1, 500, 50, 64)
    assert list(p) == g["prefix"] and [list(x) for x in items] == g["items"]
    got = w.score(g["prefix"], g["items"])
    for mode in ("naive", "ibpc", "multi_item"):
        want = np.asarray(g["modes"][mode]["scores"])
        assert np.array_equal(got, want), mode  # F8: all token modes bit-identical


def test_acceptance_criterion_1_requests_bit_exact():
    g = gold("acceptance_c1.json")
    w = port_weights(g)
    for r in g["requests"]:
        assert np.array_equal(w.score(r["prefix"], r["items"]), np.asarray(r["multi_item"]))


def test_ragged_requests_and_small_engine_config_bit_exact():
    for name, n_tasks in (("toy_ragged.json", 6), ("engine_small.json", 3)):
        g = gold(name)
        w = port_weights(g)
        for r in g["requests"]:
            mi = r["multi_item"]
            want = np.asarray(mi if isinstance(mi, list) else mi["scores"])
            got = w.score(r["prefix"], r["items"], n_tasks=n_tasks)
            assert np.array_equal(got, want), name
            for mode in ("naive", "ibpc"):  # modes are bit-identical in the reference
                if mode in r:
                    assert np.array_equal(np.asarray(r[mode]["scores"]), want)


def test_mixed_mode_bit_exact_and_equivalence():
    g = gold("mixed_c1.json")
    w = port_weights(g)
    tok = w.tensors()["tok_emb"].reshape(300, 64)
    rows = [tok[np.asarray(t)] for t in g["items"]]
    mixed = w.score(g["prefix"], rows=rows)
    assert np.array_equal(mixed, np.asarray(g["mixed_substitute"]))
    # acceptance criterion 4 (acceptance_main.cpp:146-174): mixed == ibpc within 1e-6
    assert np.abs(mixed - np.asarray(g["ibpc"])).max() <= 1e-6
    one = w.score(g["prefix"], rows=[tok[np.asarray(t[:1])] for t in g["items"]])
    assert np.array_equal(one, np.asarray(g["one_token"]))
    assert g["one_token_kv"] == 1.0


def test_attention_kat_bit_exact():
    g = gold("attention_kat.json")
    q, k, v = (np.asarray(g[x], np.float32) for x in "qkv")
    n = q.shape[0]
    sp = np.asarray(g["spans"], np.int32).reshape(-1)
    out = np.zeros_like(q)
    O.port().or_attention(q.ctypes.data_as(O.f32p), k.ctypes.data_as(O.f32p),
                          v.ctypes.data_as(O.f32p), out.ctypes.data_as(O.f32p), n, g["heads"],
                          g["head_dim"], sp.ctypes.data_as(O.i32p))
    assert np.array_equal(out, np.asarray(g["out"], np.float32))
    # dense double-precision oracle (test_kernels.cpp:106-136), rel 1e-4
    H, dh = g["heads"], g["head_dim"]
    for i, (pe, ss, pos) in enumerate(g["spans"]):
        allowed = list(range(pe)) + list(range(ss, pos + 1))
        for h in range(H):
            s = np.array([q[i, h * dh:(h + 1) * dh].astype(np.float64) @ k[a, h * dh:(h + 1) * dh]
                          for a in allowed]) / np.sqrt(dh)
            p = np.exp(s - s.max())
            p /= p.sum()
            ref = p @ v[allowed, h * dh:(h + 1) * dh].astype(np.float64)
            np.testing.assert_allclose(out[i, h * dh:(h + 1) * dh], ref, rtol=1e-4, atol=1e-6)


def test_c2_scale_bit_exact():
    """C2 dims (L20 d1024 H8 ff1536), fan-in weights, 4 items: port == reference."""
    g = gold("c2_subset.json")
    w = port_weights(g, 1)
    got = w.score(g["prefix"], g["items"], threads=0)
    assert np.array_equal(got, np.asarray(g["multi_item"]))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_port_vs_reference_fuzz(tmp_path):
    """Random configs/requests: the C restatement equals the compiled reference."""
    rng = np.random.default_rng(5)
    for trial in range(4):
        c = {"n_layers": int(rng.integers(1, 3)), "d_model": int(rng.choice([16, 32, 64])),
             "n_heads": 2, "d_ff": int(rng.choice([32, 64])), "vocab_size": 300,
             "max_seq": 512, "heads": ["a", "b"]}
        cfg = Cfg(c)
        path = str(tmp_path / f"w{trial}.srnk")
        O.ref_init_save(cfg, trial, path, fan_in=bool(trial % 2))
        w = O.OracleWeights.load(path, cfg)
        p, items = random_request(Rng(trial), int(rng.integers(0, 40)), 20, 6)
        for mode in (0, 1, 2):
            want, _, _ = O.ref_score(path, mode, p, items=items, n_tasks=3)
            assert np.array_equal(w.score(p, items, n_tasks=3), want), (trial, mode)


# ------------------------------------------------------------ retrieval scan
def test_retrieval_oracle_matches_reference_golden():
    """The C restatement of exhaustive_topk is bit-identical to the
    reference's outputs (tests/golden/retrieval.json)."""
    from tests.retrieval_cases import golden_cases
    for c in golden_cases():
        ids, sc = O.oracle_topk(c["emb"], c["feat"], c["ids"], c["keep"], c["query"], c["w0"],
                                c["w"], c["k"])
        assert np.array_equal(ids, c["ref_ids"])
        assert np.array_equal(sc, c["ref_scores"])


def test_retrieval_oracle_error_rules():
    import pytest as _pt
    from tests.retrieval_cases import random_corpus
    emb, feat, ids, _ = random_corpus(3, 50, 8, 2)
    with _pt.raises(O.RetrievalError) as e:
        O.oracle_topk(emb, feat, ids, None, emb[0], 1.0, [0.1, 0.2], 0)
    assert e.value.code == 3  # SpecViolation (retrieval.cpp:138-140)
    with _pt.raises(O.RetrievalError) as e:
        O.oracle_topk(emb, feat, ids, None, emb[0], 1.0, [0.1], 5)
    assert e.value.code == 6  # Alignment (:62-65)
    with _pt.raises(O.RetrievalError) as e:
        O.oracle_topk(emb, feat, ids, None, np.zeros(8, np.float32), 1.0, [0.1, 0.2], 5)
    assert e.value.code == 9  # DegenerateInput (:52-54)
    # no candidates: no per-candidate checks run, empty result
    ids_o, _ = O.oracle_topk(emb, feat, ids, np.zeros(50, np.uint8), np.zeros(8, np.float32), 1.0,
                             [0.1], 5)
    assert len(ids_o) == 0


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_retrieval_oracle_fuzz_against_reference():
    from tests.retrieval_cases import random_corpus
    rng = np.random.default_rng(77)
    for t in range(8):
        n, d, f = int(rng.integers(1, 3000)), int(rng.integers(1, 40)), int(rng.integers(0, 3))
        emb, feat, ids, color = random_corpus(100 + t, n, d, f, unit=bool(t % 2))
        q = rng.standard_normal(d).astype(np.float32)
        w = list(rng.standard_normal(f))
        k = int(rng.integers(1, 60))
        allowed = [int(rng.integers(0, 3))] if t % 3 == 0 else None
        keep = None if allowed is None else np.isin(color, allowed).astype(np.uint8)
        a = O.oracle_topk(emb, feat, ids, keep, q, 0.7, w, k)
        b = O.ref_topk(emb, feat, ids, color, q, 0.7, w, allowed, k)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_calibration_oracle_matches_reference_golden():
    """calibrate (calibration.cpp:65-88) restated in C == the reference's values."""
    with open(os.path.join(os.path.dirname(__file__), "golden", "calibration.json")) as f:
        g = json.load(f)
    F = lambda k: np.array([float(x) for x in g[k]])
    got = O.oracle_final_scores(F("raws")[:, None], F("lo"), F("hi"), F("value"))
    assert np.array_equal(got, F("calibrated"))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_wire_golden_reproduces_on_reference():
    """tests/golden/wire_b64.json is what the reference's decode_f32_base64 says."""
    import base64 as b64
    with open(os.path.join(os.path.dirname(__file__), "golden", "wire_b64.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        out, st, msg = O.ref_decode_f32_base64(c["text"])
        assert (st, msg) == (c["status"], c["message"])
        if st == 0:
            assert np.array_equal(out, np.frombuffer(b64.b64decode(c["floats"]), np.float32))


def test_wire_golden_valid_payloads_are_standard_base64():
    import base64 as b64
    with open(os.path.join(os.path.dirname(__file__), "golden", "wire_b64.json")) as f:
        cases = json.load(f)["cases"]
    for c in cases:
        if c["status"] == 0 and c["text"]:
            want = np.frombuffer(b64.b64decode(c["floats"]), np.float32)
            assert np.array_equal(np.frombuffer(b64.b64decode(c["text"]), np.float32), want)
