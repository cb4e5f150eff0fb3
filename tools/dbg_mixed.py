import sys, json, numpy as np
sys.path.insert(0, '.')
import paper_2602_07309_b200 as sr
from tests.test_gpu_parity import gold, cfg_of, request
g = gold("mixed_c1.json"); cfg = cfg_of(g["config"])
eng = sr.ScoringEngine(sr.init_model(cfg, 2026))
tok = sr.init_model(cfg, 2026).tensors()["tok_emb"].reshape(cfg.vocab_size, cfg.d_model)
rows = [tok[np.asarray(t)] for t in g["items"]]
ref = np.asarray(g["ibpc"])
mix = request(g["prefix"], None, sr.ScoreMode.Mixed, rows=rows)
ib = request(g["prefix"], g["items"], sr.ScoreMode.Ibpc)
print("ibpc ", [round(float(np.abs(eng.score(ib).scores - ref).max()), 6) for _ in range(4)])
print("mixed", [round(float(np.abs(eng.score(mix).scores - ref).max()), 6) for _ in range(4)])
h1 = eng.item_hidden(mix); h2 = eng.item_hidden(mix); h3 = eng.item_hidden(ib)
print("hidden mixed-vs-mixed", np.abs(h1 - h2).max(), "mixed-vs-ibpc", np.abs(h1 - h3).max())
