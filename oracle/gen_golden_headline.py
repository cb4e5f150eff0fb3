#!/usr/bin/env python3
"""Full-request golden vectors at the BASELINE.json configurations.
TEST INFRASTRUCTURE ONLY; run here, where /root/reference exists:

    make -C oracle && nice python oracle/gen_golden_headline.py [names...]

Every fixture holds, for every item of the request, the scores of
  ref32 : THE REFERENCE ITSELF (oracle/_ref = /root/reference/proj sources
          compiled in place) on the fp32 fan-in weights, in the reference's own
          mode for the request (score_multi_item_chunked, engine.cpp:328-377, or
          score_mixed, engine.cpp:238-276), and
  ref16 : the C restatement (oracle/semrank_oracle.c, pinned bit-identical to
          the reference by tests/test_oracle.py) on the same weights with the
          GEMM matrices rounded to bf16, i.e. the reference algorithm on the
          weights the device actually multiplies with.
plus the oracle's top-10 (score desc, item index asc — semrank_main.cpp:393-398).

Requests are regenerated from numpy seeds on the GPU box (bench.py's
make_request streams); a sha256 of the regenerated inputs is stored and the
tests check it before comparing. Weights are never stored: the product's
init_model(cfg, 2026, "fan_in") is byte-identical to the reference harness's
(tests/test_host.py), so the box rebuilds them.

Fixtures (tests/golden/headline_*.npz + headline.json):
  c2      configs[1]: 1 query x 256 items x 96 tokens, T_q 256 (bench seed 7)
  c3      configs[2]: 1 query x 1024 items x 8 soft-token rows (bench seed 7)
  c3proj  configs[2] with the device projection: 256 items, d_emb 256 embedding
          -> 8 soft rows through a fixed [256 x 8192] projection applied to
          bf16-rounded operands (the pre-step both sides share)
  pad     service mixed form (service.cpp:208-217): d_emb 32 retrieval
          embedding zero-padded into one d_model row, 256 items, C2 model
  c4      configs[3]: L28 d2048 H16 ff6144, query 0 of the bench batch, first
          32 of its 250 items, all 28 layers
  batch   2 queries in one pass (plan_batches generalisation), C2 model, ragged
  ragged  C2 model, one query whose items straddle the 128-row attention tiles
          (lengths 1 ... 400, prefix 100)
  ragged_soft  C2 model, mixed mode with 1 ... 20 soft rows per item
  c5      configs[4]: 1 query x 8192 items (C2 model); ref16 for all 8192,
          ref32 for a 128-item random subset
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from oracle.gen_golden import Cfg  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
TMP = os.path.join(tempfile.gettempdir(), "golden_headline")
THREADS = os.cpu_count() or 1
C2 = dict(n_layers=20, d_model=1024, n_heads=8, d_ff=1536)
C4 = dict(n_layers=28, d_model=2048, n_heads=16, d_ff=6144)


from tests.headline_inputs import (bf16, batch_requests, emb_request, pad_rows,  # noqa: E402,F401
                                    project_rows, projection_matrix, ragged_long_request,
                                    ragged_soft_request, sha, soft_request, tokens_request)


# ------------------------------------------------------------------ oracles
_weights = {}


def weights(dims, seed=2026):
    cfg = Cfg(**dims)
    key = (tuple(sorted(dims.items())), seed)
    if key not in _weights:
        os.makedirs(TMP, exist_ok=True)
        path = os.path.join(TMP, f"w_{dims['n_layers']}_{dims['d_model']}_{seed}.srnk")
        if not os.path.exists(path):
            O.ref_init_save(cfg, seed, path, fan_in=True)
        with open(path, "rb") as f:
            digest = hashlib.sha256(f.read()).hexdigest()
        _weights[key] = (cfg, path, digest)
    return _weights[key]


_port16 = {}


def port16(path):
    if path not in _port16:
        _port16.clear()
        w = O.OracleWeights.load(path)
        w.round_bf16()
        _port16[path] = w
    return _port16[path]


def ref32(path, prefix, items=None, rows=None):
    O.ref().ref_set_parallel(1)
    mode = 3 if rows is not None else 2
    s, fl, kv = O.ref_score(path, mode, prefix, items=None if items is None else list(items),
                            rows=None if rows is None else list(rows))
    return s, fl


def ref16(path, prefix, items=None, rows=None, chunk=None):
    w = port16(path)
    seq = items if items is not None else rows
    n = len(seq)
    chunk = chunk or n
    out = []
    for lo in range(0, n, chunk):
        sl = seq[lo:lo + chunk]
        out.append(w.score(prefix, items=list(sl) if items is not None else None,
                           rows=list(sl) if rows is not None else None, threads=THREADS))
    return np.concatenate(out)


def top10(s):
    rel = s[:, 0]
    return sorted(range(len(rel)), key=lambda i: (-rel[i], i))[:10]


def save(name, meta, **arrays):
    np.savez_compressed(os.path.join(GOLD, f"headline_{name}.npz"), **arrays)
    idx_path = os.path.join(GOLD, "headline.json")
    idx = {}
    if os.path.exists(idx_path):
        with open(idx_path) as f:
            idx = json.load(f)
    idx[name] = meta
    with open(idx_path, "w") as f:
        json.dump(idx, f, indent=1, sort_keys=True)
    print(f"[{time.strftime('%H:%M:%S')}] wrote headline_{name}", flush=True)


def common_meta(cfg, digest, pins):
    return {"config": cfg.as_dict(), "seed": 2026, "init": "fan_in", "weights_sha256": digest,
            "pins": pins}


# ----------------------------------------------------------------- fixtures
def gen_c2():
    cfg, path, dg = weights(C2)
    prefix, toks = tokens_request(7, 256, 96, 256)
    s32, fl = ref32(path, prefix, items=toks)
    s16 = ref16(path, prefix, items=toks)
    save("c2", {**common_meta(cfg, dg, "engine.cpp:186-236,328-377 (score_multi_item_chunked)"),
                "request": "bench.make_request c2, numpy default_rng(7)", "t_q": 256, "t_i": 96,
                "n_items": 256, "inputs_sha256": sha(prefix, toks), "flops": fl.tolist(),
                "top10_ref32": top10(s32), "top10_ref16": top10(s16)},
         ref32=s32, ref16=s16)


def gen_c3():
    cfg, path, dg = weights(C2)
    prefix, rows = soft_request(7, 256, 8, 1024, 1024)
    s32, fl = ref32(path, prefix, rows=rows)
    s16 = ref16(path, prefix, rows=rows)
    save("c3", {**common_meta(cfg, dg, "engine.cpp:238-276 (score_mixed)"),
                "request": "bench.make_request c3, numpy default_rng(7)", "t_q": 256,
                "n_soft": 8, "n_items": 1024, "inputs_sha256": sha(prefix, rows),
                "flops": fl.tolist(), "top10_ref32": top10(s32), "top10_ref16": top10(s16)},
         ref32=s32, ref16=s16)


def gen_c3proj():
    cfg, path, dg = weights(C2)
    prefix, emb = emb_request(17, 256, 256, 256)
    proj = projection_matrix(2027, 256, 8, 1024)
    rows = project_rows(emb, proj, 8, 1024)
    s32, fl = ref32(path, prefix, rows=rows)
    s16 = ref16(path, prefix, rows=rows)
    save("c3proj", {**common_meta(cfg, dg, "engine.cpp:238-276 on projected rows (SURVEY H7)"),
                    "request": "emb_request(17, 256, 256, 256), projection_matrix(2027, 256, 8, 1024)",
                    "t_q": 256, "n_soft": 8, "d_emb": 256, "n_items": 256,
                    "inputs_sha256": sha(prefix, emb, proj), "rows_sha256": sha(rows),
                    "flops": fl.tolist(), "top10_ref32": top10(s32), "top10_ref16": top10(s16)},
         ref32=s32, ref16=s16)


def gen_pad():
    cfg, path, dg = weights(C2)
    prefix, emb = emb_request(19, 256, 256, 32)
    rows = pad_rows(emb, 1024)
    s32, fl = ref32(path, prefix, rows=rows)
    s16 = ref16(path, prefix, rows=rows)
    save("pad", {**common_meta(cfg, dg, "service.cpp:208-217 + engine.cpp:238-276"),
                 "request": "emb_request(19, 256, 256, 32), zero-padded to one d_model row",
                 "t_q": 256, "d_emb": 32, "n_items": 256, "inputs_sha256": sha(prefix, emb),
                 "flops": fl.tolist(), "top10_ref32": top10(s32), "top10_ref16": top10(s16)},
         ref32=s32, ref16=s16)


def gen_c4():
    cfg, path, dg = weights(C4)
    prefix, toks = tokens_request(1000, 256, 96, 250)  # bench make_queries, query 0
    toks = toks[:32]
    s32, fl = ref32(path, prefix, items=toks)
    s16 = ref16(path, prefix, items=toks)
    save("c4", {**common_meta(cfg, dg, "model.cpp:149-352 at L28 d2048 H16 ff6144"),
                "request": "bench.make_queries c4 query 0 (numpy default_rng(1000)), first 32 items",
                "t_q": 256, "t_i": 96, "n_items": 32, "inputs_sha256": sha(prefix, toks),
                "flops": fl.tolist(), "top10_ref32": top10(s32), "top10_ref16": top10(s16)},
         ref32=s32, ref16=s16)


def gen_batch():
    cfg, path, dg = weights(C2)
    arrays, meta_q = {}, []
    for q, (prefix, items) in enumerate(batch_requests()):
        s32, fl = ref32(path, prefix, items=items)
        s16 = ref16(path, prefix, items=items)
        arrays[f"ref32_{q}"], arrays[f"ref16_{q}"] = s32, s16
        meta_q.append({"t_q": len(prefix), "n_items": len(items),
                       "inputs_sha256": sha(prefix, *items), "top10_ref16": top10(s16),
                       "top10_ref32": top10(s32)})
    save("batch", {**common_meta(cfg, dg, "engine.cpp:278-326 generalised: 2 queries, one pass"),
                   "request": "batch_requests(): numpy default_rng(23)", "queries": meta_q},
         **arrays)


def gen_ragged():
    cfg, path, dg = weights(C2)
    prefix, items = ragged_long_request()
    s32, fl = ref32(path, prefix, items=items)
    s16 = ref16(path, prefix, items=items)
    save("ragged", {**common_meta(cfg, dg, "engine.cpp:186-236 with items across attention tiles"),
                    "request": "ragged_long_request(): numpy default_rng(31)", "t_q": len(prefix),
                    "lens": [len(i) for i in items], "inputs_sha256": sha(prefix, *items),
                    "flops": fl.tolist(), "top10_ref32": top10(s32), "top10_ref16": top10(s16)},
         ref32=s32, ref16=s16)


def gen_ragged_soft():
    cfg, path, dg = weights(C2)
    prefix, rows = ragged_soft_request()
    s32, fl = ref32(path, prefix, rows=rows)
    s16 = ref16(path, prefix, rows=rows)
    save("ragged_soft", {**common_meta(cfg, dg, "engine.cpp:238-276 with 1 ... 20 rows per item"),
                         "request": "ragged_soft_request(): numpy default_rng(37)",
                         "t_q": len(prefix), "counts": [len(r) for r in rows],
                         "inputs_sha256": sha(prefix, *rows), "flops": fl.tolist(),
                         "top10_ref32": top10(s32), "top10_ref16": top10(s16)},
         ref32=s32, ref16=s16)


def gen_c5():
    cfg, path, dg = weights(C2)
    prefix, toks = tokens_request(7, 256, 96, 8192)
    part = os.path.join(TMP, "c5_ref16_partial.npy")
    chunk = 512
    done = np.load(part) if os.path.exists(part) else np.zeros((0, 6))
    while len(done) < 8192:
        lo = len(done)
        s = ref16(path, prefix, items=toks[lo:lo + chunk])
        done = np.concatenate([done, s])
        np.save(part, done)
        print(f"[{time.strftime('%H:%M:%S')}] c5 ref16 {len(done)}/8192", flush=True)
    sub = np.sort(np.random.default_rng(5).permutation(8192)[:128])
    s32, fl = ref32(path, prefix, items=toks[sub])
    save("c5", {**common_meta(cfg, dg, "engine.cpp:186-236 per item; retrieval.cpp:144-165 merge"),
                "request": "bench c5: numpy default_rng(7), 8192 x 96", "t_q": 256, "t_i": 96,
                "n_items": 8192, "inputs_sha256": sha(prefix, toks),
                "ref32_subset": sub.tolist(), "top10_ref16": top10(done)},
         ref16=done, ref32_subset=s32)


GENS = {"ragged": gen_ragged, "ragged_soft": gen_ragged_soft, "c2": gen_c2, "pad": gen_pad, "batch": gen_batch, "c3proj": gen_c3proj, "c3": gen_c3,
        "c4": gen_c4, "c5": gen_c5}


def main():
    if not O.ref_available():
        sys.exit("oracle/_ref not built: run `make -C oracle` where /root/reference exists")
    names = sys.argv[1:] or list(GENS)
    for n in names:
        t0 = time.time()
        GENS[n]()
        print(f"  {n}: {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
