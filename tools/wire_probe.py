"""Where the C3 /score wire call spends its time: native parse vs the rest."""
import base64 as b64
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2602_07309_b200 as sr  # noqa: E402
from paper_2602_07309_b200 import _capi  # noqa: E402

L, d, H, ff, t_q, t_i, n_loc, soft = bench.WORKLOADS["c3"]
cfg = sr.ModelConfig(n_layers=L, d_model=d, n_heads=H, d_ff=ff,
                     head_specs=sr.ModelConfig.default_toy().head_specs)
eng = sr.ScoringEngine(sr.init_model(cfg, 2026, "fan_in"), device=0)
rng = np.random.default_rng(7)
rows = rng.standard_normal((n_loc, t_i, d)).astype(np.float32) * np.float32(0.08)
payloads = [b64.b64encode(rows[i].tobytes()).decode() for i in range(n_loc)]
raw = json.dumps({"request_id": "wire", "prefix_tokens": rng.integers(0, 256, t_q).tolist(),
                  "mode": "mixed", "items": [{"id": str(i), "embedding_b64": p}
                                             for i, p in enumerate(payloads)]}).encode()


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps * 1e3


def parse():
    h = C.c_void_p()
    _capi.lib.sr_wire_parse(raw, len(raw), 4096, C.byref(h))
    _capi.lib.sr_wire_destroy(h)


print("body MB", len(raw) / 1e6)
print("score_json ms", round(t(lambda: eng.score_json(raw, k=10)), 3))
print("sr_wire_parse ms", round(t(parse), 3))
print("bytes(raw) copy ms", round(t(lambda: bytes(bytearray(raw))), 3))
