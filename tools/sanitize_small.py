"""compute-sanitizer target: small requests through every production kernel
class — the C2-shaped model (pair GEMMs incl. residual epilogues, tcgen05
attention, LayerNorm / embed rows, score head, top-k) on token, mixed, packed
batch and projected-embedding requests, 2 layers to keep the instrumented run
short — plus the retrieval scan and the /score wire path.

  compute-sanitizer --tool memcheck python tools/sanitize_small.py
"""
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
print("tokens", res.topk)

rows = [rng.standard_normal((L, cfg.d_model)).astype(np.float32) * 0.05 for L in (8, 1, 33)]
mixed = sr.ScoreRequest(request_id="mix", prefix_tokens=prefix[:40], mode=sr.ScoreMode.Mixed,
                        items=[sr.ScoreItem(id=f"m{i}", embedding=r, n_emb_tokens=len(r))
                               for i, r in enumerate(rows)])
print("batch", [r.topk for r in eng.score_batch([req, mixed], k=2)])

d_emb, n_soft = 256, 4
eng.set_projection(rng.standard_normal((d_emb, n_soft * cfg.d_model)).astype(np.float32) * 0.02,
                   n_soft)
emb = rng.standard_normal((37, d_emb)).astype(np.float32)
print("project", eng.score_embeddings(prefix, emb, form="project", k=3).topk)
print("pad", eng.score_embeddings(prefix, emb, form="pad", k=3).topk)

n, d = 5000, 64
corpus = sr.DeviceCorpus(rng.standard_normal((n, d)).astype(np.float32),
                         rng.standard_normal((n, 2)).astype(np.float32),
                         np.arange(n, dtype=np.int64))
ids, sc = corpus.topk(rng.standard_normal(d).astype(np.float32), 1.0, [0.3, -0.2], 50)
print("retrieval", ids[:5], sc[:2])
print("ok")
