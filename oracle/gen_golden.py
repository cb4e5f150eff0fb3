#!/usr/bin/env python3
"""Generates tests/golden/*.json by running THE REFERENCE ITSELF
(oracle/_ref/libsemrank_ref.so = /root/reference/proj sources compiled in
place). Test infrastructure only; run here, where /root/reference exists:

    make -C oracle && python oracle/gen_golden.py

Each fixture records the reference file:line whose behaviour it pins.
Doubles are written with repr() so they round-trip exactly.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests.refrng import Rng, random_request, seeded_request  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
TMP = tempfile.mkdtemp(prefix="golden_")


class Cfg:
    def __init__(self, n_layers=2, d_model=64, n_heads=4, d_ff=256, vocab_size=300,
                 max_seq=4096, heads=("click", "apply", "badfit", "shortlist", "dismiss")):
        self.n_layers, self.d_model, self.n_heads, self.d_ff = n_layers, d_model, n_heads, d_ff
        self.vocab_size, self.max_seq = vocab_size, max_seq
        self.yes_token_id, self.no_token_id = 261, 262

        class H:
            def __init__(self, n):
                self.name, self.arity = n, 1
        self.head_specs = [H(n) for n in heads]

    def as_dict(self):
        return {"n_layers": self.n_layers, "d_model": self.d_model, "n_heads": self.n_heads,
                "d_ff": self.d_ff, "vocab_size": self.vocab_size, "max_seq": self.max_seq,
                "heads": [h.name for h in self.head_specs]}


def dump(name, obj):
    path = os.path.join(GOLD, name)
    with open(path, "w") as f:
        json.dump(obj, f, indent=1)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def weights(cfg, seed, fan_in=False):
    path = os.path.join(TMP, f"w_{cfg.n_layers}_{cfg.d_model}_{seed}_{int(fan_in)}.srnk")
    O.ref_init_save(cfg, seed, path, fan_in=fan_in)
    with open(path, "rb") as f:
        digest = hashlib.sha256(f.read()).hexdigest()
    return path, digest


def scores_all_modes(path, prefix, items, n_tasks):
    out = {}
    for mode, name in ((0, "naive"), (1, "ibpc"), (2, "multi_item")):
        s, fl, kv = O.ref_score(path, mode, prefix, items=items, n_tasks=n_tasks)
        out[name] = {"scores": s.tolist(), "flops": fl.tolist(), "kv_incremental_per_item": kv}
    return out


def main():
    os.makedirs(GOLD, exist_ok=True)
    if not O.ref_available():
        sys.exit("oracle/_ref not built: run `make -C oracle` where /root/reference exists")
    lib = O.ref()
    lib.ref_set_parallel(1)

    # --- RNG stream pin (rng.hpp:33-47)
    ints = O.np.zeros(16, O.np.int64)
    lib.ref_uniform_ints(101, 0, 255, 16, ints.ctypes.data_as(O.i64p))
    dump("rng_stream.json", {"pins": "include/semrank/rng.hpp:18-47", "seed": 101, "lo": 0,
                             "hi": 255, "values": ints.tolist()})

    # --- toy ranker, cmd_bench request (semrank_main.cpp:599-616), seed 1
    toy = Cfg()
    path, digest = weights(toy, 1)
    r = Rng.substream(1, "bench")
    prefix = [r.uniform_int(0, 255) for _ in range(500)]
    items = [[r.uniform_int(0, 255) for _ in range(50)] for _ in range(64)]
    dump("toy_bench.json", {
        "pins": "model.cpp:94-352, engine.cpp:100-387, semrank_main.cpp:599-616",
        "config": toy.as_dict(), "seed": 1, "init": "reference", "weights_sha256": digest,
        "request": {"stream": "substream(1,'bench')", "t_q": 500, "t_i": 50, "n_items": 64},
        "prefix": prefix, "items": items,
        "modes": scores_all_modes(path, prefix, items, 6)})

    # --- acceptance criterion 1 (acceptance_main.cpp:90-104): toy seed 2026, Rng(101), (50,150,50)
    path26, digest26 = weights(toy, 2026)
    rng = Rng(101)
    reqs = []
    for _ in range(3):
        p, its = seeded_request(rng, 50, 150, 50)
        s, fl, kv = O.ref_score(path26, 2, p, items=its, n_tasks=6)
        reqs.append({"prefix": p, "items": its, "multi_item": s.tolist(), "flops": fl.tolist()})
    dump("acceptance_c1.json", {"pins": "acceptance_main.cpp:90-104", "config": toy.as_dict(),
                                "seed": 2026, "weights_sha256": digest26, "rng_seed": 101,
                                "requests": reqs})

    # --- mixed mode (engine.cpp:238-276; acceptance_main.cpp:146-174): Rng(104), (40,12,10)
    rng = Rng(104)
    p, its = seeded_request(rng, 40, 12, 10)
    ibpc, _, _ = O.ref_score(path26, 1, p, items=its, n_tasks=6)
    tokw = np.fromfile(path26, dtype=np.uint8)  # not used: embeddings rebuilt from weights
    del tokw
    # substitute-embedding rows come from the port's (bit-identical) weights
    ow = O.OracleWeights.load(path26)
    tok = ow.tensors()["tok_emb"].reshape(300, 64)
    rows = [tok[np.asarray(t)] for t in its]
    mixed, flm, kvm = O.ref_score(path26, 3, p, rows=rows, n_tasks=6)
    one_rows = [tok[np.asarray(t[:1])] for t in its]
    one, fl1, kv1 = O.ref_score(path26, 3, p, rows=one_rows, n_tasks=6)
    dump("mixed_c1.json", {"pins": "engine.cpp:238-276, acceptance_main.cpp:146-174",
                           "config": toy.as_dict(), "seed": 2026, "rng_seed": 104,
                           "prefix": p, "items": its, "ibpc": ibpc.tolist(),
                           "mixed_substitute": mixed.tolist(), "mixed_flops": flm.tolist(),
                           "one_token": one.tolist(), "one_token_kv": kv1})

    # --- ragged toy requests (test_engine.cpp:140-162 shape, d=64 so the GPU can run it)
    path9, digest9 = weights(toy, 1234)
    rng = Rng(7)
    rr = []
    for t in range(4):
        p, its = random_request(rng, 12 + t * 3, 10, 5)
        modes = scores_all_modes(path9, p, its, 6)
        rr.append({"prefix": p, "items": its, **modes})
    dump("toy_ragged.json", {"pins": "test_engine.cpp:30-46,140-162", "config": toy.as_dict(),
                             "seed": 1234, "weights_sha256": digest9, "rng_seed": 7,
                             "requests": rr})

    # --- reference unit-test model (engine_config, test_engine.cpp:18-28): d16, hd8 (CPU only)
    small = Cfg(n_layers=2, d_model=16, n_heads=2, d_ff=32, vocab_size=264, max_seq=1024,
                heads=("click", "apply"))
    paths, digests = weights(small, 1234)
    rng = Rng(7)
    sr = []
    for t in range(6):
        p, its = random_request(rng, 12 + t * 3, 10, 5)
        s, fl, kv = O.ref_score(paths, 2, p, items=its, n_tasks=3)
        sr.append({"prefix": p, "items": its, "multi_item": s.tolist()})
    dump("engine_small.json", {"pins": "test_engine.cpp:140-162 (engine_config)",
                               "config": small.as_dict(), "seed": 1234,
                               "weights_sha256": digests, "requests": sr})

    # --- attention KAT (test_kernels.cpp:83-137): spans prefix [0,4), items [4,9), [9,12)
    H, dh, n = 2, 8, 12
    rng = np.random.default_rng(17)
    q = rng.standard_normal((n, H * dh)).astype(np.float32)
    k = rng.standard_normal((n, H * dh)).astype(np.float32)
    v = rng.standard_normal((n, H * dh)).astype(np.float32)
    spans = [[0, 0, p] for p in range(4)] + [[4, 4, p] for p in range(4, 9)] + \
            [[4, 9, p] for p in range(9, 12)]
    sp = np.asarray(spans, np.int32).reshape(-1)
    out = np.zeros((n, H * dh), np.float32)
    lib.ref_attention(q.ctypes.data_as(O.f32p), k.ctypes.data_as(O.f32p),
                      v.ctypes.data_as(O.f32p), out.ctypes.data_as(O.f32p), n, H, dh,
                      sp.ctypes.data_as(O.i32p))
    dump("attention_kat.json", {"pins": "kernels.cpp:51-95,175-192; test_kernels.cpp:83-137",
                                "heads": H, "head_dim": dh, "q": q.tolist(), "k": k.tolist(),
                                "v": v.tolist(), "spans": spans, "out": out.tolist()})

    # --- flops + plan_batches (engine.cpp:30-88, 278-326)
    fl = []
    for mode, tq, ti, nn in [(0, 500, 50, 100), (1, 500, 50, 100), (0, 50, 150, 50),
                             (1, 50, 150, 50), (3, 40, 1, 8), (0, 500, 50, 0), (1, 500, 50, 0),
                             (2, 256, 96, 256)]:
        o5 = np.zeros(5)
        lib.ref_flops(mode, tq, ti, nn, o5.ctypes.data_as(O.f64p))
        fl.append({"mode": mode, "t_q": tq, "t_i": ti, "n": nn, "report": o5.tolist()})
    rng = Rng(61)
    plans = []
    for _ in range(30):
        n_req = rng.uniform_int(1, 6)
        prefixes, lens = [], []
        for _ in range(n_req):
            n_items = rng.uniform_int(1, 8)
            lens.append([rng.uniform_int(1, 30) for _ in range(n_items)])
            prefixes.append(rng.uniform_int(1, 40))
        pl = np.asarray(prefixes, np.int32)
        off = np.zeros(n_req + 1, np.int32)
        off[1:] = np.cumsum([len(x) for x in lens])
        il = np.asarray([x for l in lens for x in l], np.int32)
        outq = np.zeros(4 * 512, np.int32)
        nout = np.zeros(1, np.int32)
        tok = np.zeros(512, np.int64)
        st = lib.ref_plan_batches(n_req, pl.ctypes.data_as(O.i32p), off.ctypes.data_as(O.i32p),
                                  il.ctypes.data_as(O.i32p), 90, outq.ctypes.data_as(O.i32p), 512,
                                  nout.ctypes.data_as(O.i32p), tok.ctypes.data_as(O.i64p))
        assert st == 0
        ne = int(nout[0])
        quads = outq[:4 * ne].reshape(-1, 4).tolist()
        nb = (max(qd[0] for qd in quads) + 1) if quads else 0
        plans.append({"prefix": prefixes, "item_lens": lens, "budget": 90, "entries": quads,
                      "batch_tokens": tok[:nb].tolist()})
    dump("host_logic.json", {"pins": "engine.cpp:30-88,278-326", "flops": fl,
                             "plan_batches": plans})

    # --- C2-scale pin: fan-in weights, 4 items of the C2 shape
    c2 = Cfg(n_layers=20, d_model=1024, n_heads=8, d_ff=1536)
    pathc2, digc2 = weights(c2, 2026, fan_in=True)
    lib.ref_set_parallel(1)
    rng = Rng.substream(7, "c2")
    prefix = [rng.uniform_int(0, 255) for _ in range(256)]
    items = [[rng.uniform_int(0, 255) for _ in range(96)] for _ in range(4)]
    s, fl, kv = O.ref_score(pathc2, 2, prefix, items=items, n_tasks=6)
    dump("c2_subset.json", {"pins": "model.cpp:149-352 at C2 dims (L20 d1024 H8 ff1536)",
                            "config": c2.as_dict(), "seed": 2026, "init": "fan_in",
                            "weights_sha256": digc2, "request_stream": "substream(7,'c2')",
                            "prefix": prefix, "items": items, "multi_item": s.tolist()})


def _b64(a):
    import base64
    return base64.b64encode(np.ascontiguousarray(a).tobytes()).decode()


def retrieval():
    """exhaustive_topk cases (retrieval.cpp:134-173) from the reference, shaped
    like test_retrieval.cpp:170-255: random unit corpora with a colour
    attribute, random k and filters; tied scores; K above the corpus size."""
    rng = np.random.default_rng(20261017)
    cases = []
    for t in range(6):
        n, d, f = (400, 16, 2) if t < 4 else (257, 32, 1)
        emb = rng.standard_normal((n, d)).astype(np.float32)
        emb /= np.linalg.norm(emb, axis=1, keepdims=True).astype(np.float32)
        feat = rng.random((n, f)).astype(np.float32)
        ids = rng.permutation(n * 3)[:n].astype(np.int64)
        color = rng.integers(0, 3, n).astype(np.int32)
        q = rng.standard_normal(d).astype(np.float32)
        q /= np.float32(np.linalg.norm(q))
        k = int(rng.integers(1, 41))
        allowed = [0, 1] if t % 2 else None
        w = [0.2, -0.1][:f]
        oi, osc = O.ref_topk(emb, feat, ids, color, q, 1.0, w, allowed, k)
        cases.append({"n": n, "d": d, "f": f, "emb": _b64(emb), "feat": _b64(feat),
                      "ids": ids.tolist(), "color": color.tolist(), "query": _b64(q),
                      "w0": 1.0, "w": w, "allowed": allowed, "k": k,
                      "ref_ids": oi.tolist(), "ref_scores": [repr(float(x)) for x in osc]})
    # ties: equal scores everywhere -> ascending doc_id (test_retrieval.cpp:223-240)
    emb = np.tile(np.array([[1.0, 0.0]], np.float32), (4, 1))
    ids = np.array([3, 2, 1, 0], np.int64)
    oi, osc = O.ref_topk(emb, np.zeros((4, 0), np.float32), ids, None, np.array([1, 0], np.float32),
                         1.0, [], None, 10)
    cases.append({"n": 4, "d": 2, "f": 0, "emb": _b64(emb), "feat": "", "ids": ids.tolist(),
                  "color": None, "query": _b64(np.array([1, 0], np.float32)), "w0": 1.0, "w": [],
                  "allowed": None, "k": 10, "ref_ids": oi.tolist(),
                  "ref_scores": [repr(float(x)) for x in osc]})
    dump("retrieval.json", {"source": "exhaustive_topk retrieval.cpp:134-173 via oracle/_ref",
                            "cases": cases})


def calibration():
    """fit_isotonic + calibrate (calibration.cpp:13-88) from the reference:
    a head fitted on random (score, outcome) pairs (with ties) and calibrated
    values of raw scores below, inside, between and above its blocks."""
    rng = np.random.default_rng(20261018)
    raw = np.round(rng.random(300), 3)  # rounding makes equal-score pools
    oc = (rng.random(300) < raw).astype(np.int32)
    raws = np.concatenate([rng.random(200), raw[:20], [-0.5, 0.0, 1.0, 1.5]])
    lo, hi, val, cal = O.ref_fit_calibrate(raw, oc, raws)
    dump("calibration.json", {"source": "fit_isotonic/calibrate calibration.cpp:13-88 via oracle/_ref",
                              "lo": [repr(float(x)) for x in lo], "hi": [repr(float(x)) for x in hi],
                              "value": [repr(float(x)) for x in val],
                              "raws": [repr(float(x)) for x in raws],
                              "calibrated": [repr(float(x)) for x in cal]})


def wire():
    """decode_f32_base64 (base64.cpp:60-108) outcomes from the reference on
    well-formed payloads (every padding length) and each malformation."""
    import base64 as b64
    rng = np.random.default_rng(20261019)
    cases = []
    for n in (1, 2, 3, 16, 64):
        v = rng.standard_normal(n).astype(np.float32)
        t = b64.b64encode(v.tobytes()).decode()
        out, st, msg = O.ref_decode_f32_base64(t)
        cases.append({"text": t, "status": st, "message": msg,
                      "floats": _b64(out) if out is not None else None})
    good = b64.b64encode(rng.standard_normal(6).astype(np.float32).tobytes()).decode()
    for t in [good[:-1], "AA=A" + good[4:], good[:8] + "*" + good[9:], good[:-4] + "A=A=",
              good[:-4] + "AA=B", b64.b64encode(b"\x01\x02\x03").decode(), "", "====",
              "AAA=AAAA"]:
        out, st, msg = O.ref_decode_f32_base64(t)
        cases.append({"text": t, "status": st, "message": msg,
                      "floats": _b64(out) if out is not None else None})
    dump("wire_b64.json", {"source": "decode_f32_base64 base64.cpp:60-108 via oracle/_ref",
                           "cases": cases})


def score_cache():
    """canonical_query / fnv1a64 / ScoreCache LRU traces (midtier.cpp:14-100)
    from the reference, incl. test_midtier.cpp:18-85's cases."""
    queries = [
        ("Senior  ML Engineer ", [("region", "na"), ("region", "emea")]),
        ("senior ml engineer", [("region", "emea"), ("region", "na")]),
        ("nurse", []), ("doctor", []), ("a", [("x", "1")]), ("a", []),
        ("", []), ("   ", []), ("\tMixed\nCASE  text\r\n", []),
        ("q", [("b", "2"), ("a", "z"), ("a", "y"), ("B", "1")]),
        ("Data Scientist", [("seniority", "senior"), ("region", "us"), ("region", "apac")]),
        ("caf\u00e9 ZURICH", [("lang", "de")]),
    ]
    qcases = []
    for text, filt in queries:
        canon, h = O.ref_canonical_query(text, filt)
        qcases.append({"text": text, "filters": filt, "canonical": canon, "fnv1a64": str(h)})
    traces = []
    # test_midtier.cpp:27-56 as a script
    A, B, Cc = ("s", 1, 1, "v"), ("s", 1, 2, "v"), ("s", 1, 3, "v")
    ops = [(0,) + A + (0.0,), (1,) + A + (0.9,), (0,) + A + (0.0,), (1,) + B + (0.5,),
           (1,) + Cc + (0.1,), (0,) + A + (0.0,), (0,) + B + (0.0,), (0,) + Cc + (0.0,),
           (0,) + B + (0.0,), (1,) + A + (0.9,), (0,) + B + (0.0,), (0,) + Cc + (0.0,),
           (1,) + A + (0.9,), (1,) + A + (0.5,)]
    st, msg, out = O.ref_cache_trace(2, ops)
    traces.append({"capacity": 2, "ops": ops, "status": st, "message": msg, "out": out})
    # random traces over several key fields (searchers, signatures, versions)
    rng = np.random.default_rng(20261017)
    for cap in (1, 4, 16):
        ops = []
        for _ in range(400):
            e = int(rng.integers(0, 12))
            who = ["s", "t"][int(rng.integers(0, 2))]
            sig = [7, 2**63 + 5][int(rng.integers(0, 2))]
            ver = ["v", "w"][int(rng.integers(0, 2))]
            ops.append((int(rng.integers(0, 2)), who, sig, e, ver, float(e) + 0.25 * len(who + ver)))
        st, msg, out = O.ref_cache_trace(cap, ops)
        traces.append({"capacity": cap, "ops": ops, "status": st, "message": msg, "out": out})
    st, msg, _ = O.ref_cache_trace(0, [])
    dump("score_cache.json", {"source": "canonical_query/fnv1a64/ScoreCache midtier.cpp:14-100 "
                                        "via oracle/_ref", "queries": qcases, "traces": traces,
                              "zero_capacity": {"status": st, "message": msg}})


def text_api():
    """build_prompt (prompt.cpp:14-38) and score_result_to_json
    (service.cpp:380-391) outputs from the reference: prompt splits incl. both
    error rules, and response bodies over random probabilities, exact binary
    fractions, integers, tiny/huge magnitudes, -0.0 and ids that need escaping."""
    prompts = []
    for sysm, q, doc, ms in [(b"You rank jobs.\n", b"query: nurse", b"RN, night shift", 4096),
                             (b"", b"q", b"", 4096), (b"S", b"", b"doc", 4096),
                             (b"", b"", b"doc", 4096), (b"abc", b"def", b"g" * 10, 29),
                             (b"abc", b"def", b"g" * 10, 30), (b"", b"", b"", 4096),
                             ("caf\u00e9 \u2603".encode(), b"\x01\xff", b"\x7fx", 64)]:
        st, msg, pre, item = O.ref_build_prompt(sysm, q, doc, ms)
        prompts.append({"system": _b64(np.frombuffer(sysm, np.uint8)) if sysm else "",
                        "query": _b64(np.frombuffer(q, np.uint8)) if q else "",
                        "document": _b64(np.frombuffer(doc, np.uint8)) if doc else "",
                        "max_seq": ms, "status": st, "message": msg, "prefix": pre, "item": item})
    rng = np.random.default_rng(20261020)
    names = [b"relevance", b"click", b"apply", b"badfit", b"shortlist", b"dismiss"]
    specials = [0.0, -0.0, 1.0, 0.5, 0.1, 1e-5, 1.5e-4, 0.00012345, 1e15, 123456789012345.0,
                1234567890123456.0, 1e16, 1.5e20, 2.0 ** -1074, 1.7976931348623157e308,
                0.3333333333333333, 2.0 / 3.0, 100.0, 15007744.0, 5e-324, 9.999999999999999e-5,
                1e-4, 1e21, 123.456, -2.5e-7]
    bodies = []
    for t in range(6):
        n = int(rng.integers(0, 9))
        ids = [str(int(rng.integers(0, 10**6))).encode() for _ in range(n)]
        if t == 3 and n:
            ids[0] = 'a"b\\c\n\t\x01\x1f\u00e9\u2603/'.encode()
        if t % 2:
            sc = rng.random((n, len(names)))
        else:
            sc = rng.choice(specials, (n, len(names)))
        att, lin = (float(rng.integers(0, 10**8)), float(rng.random() * 1e6)) if t else (0.0, 5e-5)
        rid = (b"req-%d" % t) if t != 5 else "r\u00e9q\"x\"".encode()
        st, msg, body = O.ref_score_result_json(rid, ids, names, sc, att, lin)
        assert st == 0, msg
        bodies.append({"request_id": _b64(np.frombuffer(rid, np.uint8)),
                       "ids": [_b64(np.frombuffer(i, np.uint8)) if i else "" for i in ids],
                       "names": [x.decode() for x in names],
                       "scores": [[repr(float(v)) for v in row] for row in sc],
                       "attention": repr(att), "linear": repr(lin), "json": body.decode()})
    # every special value and 2000 random doubles of all magnitudes, one per item
    vals = specials + [float(x) for x in rng.random(1000)] + \
        [float(np.ldexp(rng.random(), int(e))) for e in rng.integers(-60, 80, 1000)]
    bits = rng.integers(0, 0x7FF0000000000000, 3000, dtype=np.int64)  # any finite double
    vals += [float(x) for x in bits.view(np.float64)]
    ids = [str(i).encode() for i in range(len(vals))]
    st, msg, body = O.ref_score_result_json(b"nums", ids, [b"relevance"],
                                            np.asarray(vals)[:, None], 1.0, 2.0)
    bodies.append({"request_id": _b64(np.frombuffer(b"nums", np.uint8)),
                   "ids": [_b64(np.frombuffer(i, np.uint8)) for i in ids], "names": ["relevance"],
                   "scores": [[repr(v)] for v in vals], "attention": "1.0", "linear": "2.0",
                   "json": body.decode()})
    dump("text_api.json", {"source": "build_prompt prompt.cpp:14-38 and score_result_to_json "
                                     "service.cpp:380-391 via oracle/_ref",
                           "prompts": prompts, "bodies": bodies})


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "text_api":
        text_api()
    elif len(sys.argv) > 1 and sys.argv[1] == "score_cache":
        score_cache()
    elif len(sys.argv) > 1 and sys.argv[1] == "wire":
        wire()
    elif len(sys.argv) > 1 and sys.argv[1] == "calibration":
        calibration()
    elif len(sys.argv) > 1 and sys.argv[1] == "retrieval":
        if not O.ref_available():
            sys.exit("oracle/_ref not built")
        retrieval()
    else:
        main()
        retrieval()
        calibration()
        wire()
        score_cache()
        text_api()
