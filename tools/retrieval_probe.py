"""Per-call host/device split of the 200k-doc retrieval query."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_07309_b200.retrieval import DeviceCorpus  # noqa: E402

n, d, f, k = bench.RETRIEVAL["retrieval"]
emb, feat, ids = bench.make_corpus(n, d, f)
corpus = DeviceCorpus(emb, feat, ids)
q = np.random.default_rng(11).standard_normal(d).astype(np.float32)
w = [0.3] * f
for _ in range(20):
    corpus.topk(q, 0.9, w, k)
torch.cuda.synchronize()
reps = int(os.environ.get("REPS", "200"))
t = time.perf_counter()
for _ in range(reps):
    corpus.topk(q, 0.9, w, k)
dt = (time.perf_counter() - t) / reps * 1e3
print(f"topk ms {dt:.4f} scan ms {corpus.last_scan_ms():.4f} candidates {corpus.last_candidates()}")

import ctypes as C  # noqa: E402
from paper_2602_07309_b200 import _capi  # noqa: E402
qq = np.ascontiguousarray(q)
wv = np.ascontiguousarray(w, dtype=np.float64)
oi = np.zeros(k, np.int64)
osc = np.zeros(k, np.float64)
nn = C.c_int32(0)
args = (corpus._h, qq.ctypes.data, d, 0.9, wv.ctypes.data, len(wv), None, k,
        oi.ctypes.data_as(C.POINTER(C.c_int64)), osc.ctypes.data_as(C.POINTER(C.c_double)), C.byref(nn))
fn = _capi.lib.sr_corpus_topk
t = time.perf_counter()
for _ in range(reps):
    fn(*args)
print(f"raw sr_corpus_topk ms {(time.perf_counter() - t) / reps * 1e3:.4f}")
ev = torch.cuda.Event()
t = time.perf_counter()
for _ in range(reps):
    ev.record()
    ev.synchronize()
print(f"event record+sync ms {(time.perf_counter() - t) / reps * 1e3:.4f}")
