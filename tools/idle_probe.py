"""Serving diagnostic: wall time of one C2 scoring call (public API, host
arrays) after the device sat idle for X ms, to see whether sporadic slow
passes at light load come from the idle gap before them."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_07309_b200 as sr  # noqa: E402

cfg = sr.ModelConfig(n_layers=20, d_model=1024, n_heads=8, d_ff=1536,
                     head_specs=sr.ModelConfig.default_toy().head_specs)
eng = sr.ScoringEngine(sr.init_model(cfg, 2026, "fan_in"), device=0)
rng = np.random.default_rng(7)
prefix = rng.integers(0, 256, 256).astype(np.int32)
toks = rng.integers(0, 256, (256, 96)).astype(np.int32)
req = sr.ScoreRequest(request_id="c2", prefix_tokens=prefix, mode=sr.ScoreMode.MultiItem,
                      items=[sr.ScoreItem(id=str(i), tokens=t) for i, t in enumerate(toks)])
for _ in range(5):
    eng.score(req, k=10)
for idle_ms in [0, 0, 10, 30, 60, 100, 200, 400, 800, 1600] * 3:
    time.sleep(idle_ms / 1000.0)
    t0 = time.perf_counter()
    eng.score(req, k=10)
    t1 = time.perf_counter()
    t2 = time.perf_counter()
    eng.score(req, k=10)
    t3 = time.perf_counter()
    print(f"idle {idle_ms:5d} ms: first call {1e3 * (t1 - t0):7.2f} ms, next {1e3 * (t3 - t2):7.2f} ms",
          flush=True)
