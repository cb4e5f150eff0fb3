"""GPU diagnostic: engine vs oracle(bf16 weights) deviation across model dims."""
import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_07309_b200 as sr
from oracle import oracle as O
heads = sr.ModelConfig.default_toy().head_specs
cases = [
  (1, 1024, 8, 1536, 256, [96]*5),
  (1, 1024, 8, 1536, 64, [32]*2),
  (1, 256, 2, 256, 64, [32]*2),
  (1, 128, 1, 128, 64, [32]*2),
  (1, 128, 8, 128, 64, [32]*2),
  (1, 64, 4, 256, 64, [32]*2),
  (1, 64, 1, 64, 64, [32]*2),
  (1, 512, 8, 512, 64, [32]*2),
  (2, 1024, 8, 1536, 256, [96]*5),
]
for L, d, H, F, tq, lens in cases:
    cfg = sr.ModelConfig(n_layers=L, d_model=d, n_heads=H, d_ff=F, head_specs=heads)
    w = sr.init_model(cfg, 2026, "fan_in")
    rng = np.random.default_rng(7)
    prefix = [int(x) for x in rng.integers(0, 256, tq)]
    items = [[int(x) for x in rng.integers(0, 256, n)] for n in lens]
    ow = O.OracleWeights.init(cfg, 2026, 1); ow.cfg = O.config_struct(cfg); ow.round_bf16()
    s_ref, h_ref = ow.score(prefix, items, hidden=True)
    eng = sr.ScoringEngine(w)
    req = sr.ScoreRequest(prefix_tokens=prefix, items=[sr.ScoreItem(id=str(i), tokens=t) for i, t in enumerate(items)], mode=sr.ScoreMode.MultiItem)
    res = eng.score(req)
    hid = eng.item_hidden(req)
    print(f"L{L} d{d} H{H} hd{d//H} F{F} tq{tq} lens{lens[:2]}: score dev {np.abs(res.scores - s_ref).max():.3e}  hidden dev {np.abs(hid-h_ref).max():.3e} (|h| {np.abs(h_ref).max():.2f})", flush=True)
