"""Kernel-variant bit-identity aid: scores of the C2 request (seed 7) and of a
ragged token request (item lengths 1..400, items straddling attention tiles)
from the library SEMRANK_LIB selects, written to argv[1] (.npz). Two dumps
from two builds compare with `python tools/scores_dump.py --cmp a.npz b.npz`."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    if sys.argv[1] == "--cmp":
        a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
        for k in a.files:
            same = np.array_equal(a[k], b[k])
            print(k, "bit-identical" if same else f"DIFFERS max |d| {np.abs(a[k] - b[k]).max():.3e}")
        sys.exit(0 if all(np.array_equal(a[k], b[k]) for k in a.files) else 1)
    import paper_2602_07309_b200 as sr
    cfg = sr.ModelConfig(n_layers=20, d_model=1024, n_heads=8, d_ff=1536,
                         head_specs=sr.ModelConfig.default_toy().head_specs)
    eng = sr.ScoringEngine(sr.init_model(cfg, 2026, "fan_in"), device=0)
    out = {}
    rng = np.random.default_rng(7)
    prefix = rng.integers(0, 256, 256).astype(np.int32)
    toks = rng.integers(0, 256, (256, 96)).astype(np.int32)
    req = sr.ScoreRequest(request_id="c2", prefix_tokens=prefix, mode=sr.ScoreMode.MultiItem,
                          items=[sr.ScoreItem(id=str(i), tokens=t) for i, t in enumerate(toks)])
    out["c2"] = eng.score(req, k=10).scores
    rng = np.random.default_rng(11)
    lens = rng.integers(1, 401, 48)
    items = [rng.integers(0, 256, int(n)).astype(np.int32) for n in lens]
    req = sr.ScoreRequest(request_id="ragged", prefix_tokens=prefix[:200], mode=sr.ScoreMode.MultiItem,
                          items=[sr.ScoreItem(id=str(i), tokens=t) for i, t in enumerate(items)])
    out["ragged"] = eng.score(req, k=10).scores
    np.savez(sys.argv[1], **out)
    print("wrote", sys.argv[1], {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
