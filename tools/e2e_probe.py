"""Where an end-to-end call spends its time (host packing vs device):

  REPS=200 python tools/e2e_probe.py c1
"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2602_07309_b200 as sr  # noqa: E402
from paper_2602_07309_b200 import semrank as S  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
L, d, H, ff, t_q, t_i, n_loc, soft = bench.WORKLOADS[wl]
cfg = sr.ModelConfig(n_layers=L, d_model=d, n_heads=H, d_ff=ff,
                     head_specs=sr.ModelConfig.default_toy().head_specs)
eng = sr.ScoringEngine(sr.init_model(cfg, 2026, "fan_in"), device=0)
req, ids = bench.make_request(sr, wl, 1, 0)


REPS = int(os.environ.get("REPS", "10"))


def t(fn, reps=REPS):
    fn()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - a) / reps * 1e3


print("score() ms", round(t(lambda: eng.score(req, 10)), 3))
print("pack ms", round(t(lambda: S._PackedRequest(req, d)), 3))
pr = S._PackedRequest(req, d)
rb = S._ResultBuf(len(req.items), len(eng.task_names), 10)
print("sr_engine_score ms", round(t(lambda: S._check(S._lib.sr_engine_score(eng._h, C.byref(pr.c), C.byref(rb.c)))), 3))
print("to_result ms", round(t(lambda: eng._to_result(req, rb)), 3))
plan = eng.plan(req, 10)
print("plan run (device) ms", round(t(lambda: (plan.run(), plan.sync())), 3))
print("plan fetch ms", round(t(lambda: plan.fetch()), 3))
print("python pack+resbuf+result ms", round(t(lambda: (S._PackedRequest(req, d),
                                                       S._ResultBuf(len(req.items), len(eng.task_names), 10),
                                                       eng._to_result(req, rb))), 3))
