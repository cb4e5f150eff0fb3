"""compute-sanitizer target: one small request through every production
kernel class of the C2 model (pair GEMMs incl. residual epilogues, tcgen05
attention, LayerNorm / embed rows, score head, top-k), 2 layers to keep the
instrumented run short."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_07309_b200 as sr  # noqa: E402

cfg = sr.ModelConfig(n_layers=2, d_model=1024, n_heads=8, d_ff=1536,
                     head_specs=sr.ModelConfig.default_toy().head_specs)
eng = sr.ScoringEngine(sr.init_model(cfg, 2026, "fan_in"), device=0)
rng = np.random.default_rng(3)
prefix = rng.integers(0, 256, 256).astype(np.int32)
req = sr.ScoreRequest(request_id="san", prefix_tokens=prefix, mode=sr.ScoreMode.MultiItem,
                      items=[sr.ScoreItem(id=str(i), tokens=rng.integers(0, 256, L).astype(np.int32))
                             for i, L in enumerate([96, 7, 130, 1, 96, 64])])
res = eng.score(req, k=3)
print("ok", res.topk)
