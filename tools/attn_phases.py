"""GPU tuning aid: per-phase softmax timeline of blocks 8..15 of the
attention kernel (library built with -DSRK_ATTN_PHASES -DSRK_TRACE_STRIDE=128,
selected with SEMRANK_LIB). Phases: S seen, TMEM loaded, max, pair exchange,
rescale check, exponentials, P stored."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07309_b200._capi import lib  # noqa: E402

H, hd, tq, L, n = 8, 128, 256, 96, 256
spans = [[0, 0, 0, 0]] * tq
cur = tq
for _ in range(n):
    spans += [[0, tq, cur, 0]] * L
    cur += L
M = len(spans)
d = H * hd
dev = torch.device("cuda:0")
qkv = (torch.randn(M, 3 * d, device=dev) * 0.5).bfloat16()
out = torch.zeros(M, d, dtype=torch.bfloat16, device=dev)
sp = np.asarray(spans, np.int32).reshape(-1)
trace = torch.zeros(256 * 256, dtype=torch.int64, device=dev)
for it in range(3):
    if it == 2:
        assert lib.sr_debug_attention_trace(C.c_void_p(trace.data_ptr())) == 0
    assert lib.sr_kernel_attention(C.c_void_p(qkv.data_ptr()),
                                   sp.ctypes.data_as(C.POINTER(C.c_int32)), M, H, hd,
                                   C.c_void_p(out.data_ptr()), None) == 0, lib.sr_last_error()
torch.cuda.synchronize()
lib.sr_debug_attention_trace(None)
t = trace.view(256, 256).cpu().numpy().astype(np.int64)
names = ["ld", "max", "xchg", "resc", "exp", "st"]
for b in [0, 77, 147]:
    row = t[b]
    print(f"cta {b}: end {int(row[29] - row[0])}")
    for g in range(8, 16):
        s0 = row[1 + g]
        ph = [int(row[64 + 16 * (g - 8) + k] - s0) for k in range(6)]
        pd = int(row[32 + g] - s0)
        nxt = int(row[1 + g + 1] - row[32 + g]) if g + 1 < 24 else -1
        q = lambda k: int(row[64 + 16 * (g - 8) + k] - s0)
        print(f"  g{g} @{int(s0 - row[0])}: " + " ".join(f"{nm}+{v}" for nm, v in zip(names, ph)) +
              f" done+{pd} nextS {nxt} | quads st {q(13)} {q(14)} {q(15)} slice1 {q(9)} | mma: S_iss {q(6)} P_seen {q(8)} PV_iss {q(7)}"
              f" | tma: K_ld {q(10)} V_ld {q(11)}")
    for li in range(8):
        q = lambda k: int(row[192 + 8 * li + k] - row[0]) if row[192 + 8 * li + k] else -1
        print(f"  item {li}: epi l_ready {q(0)} o_full {q(1)} q_empty {q(2)} | Q load {q(3)} | "
              f"MMA q_full {q(4)} | softmax S0 {q(5)}")
ends = t[:148, 29] - t[:148, 0]
print("cta cycles: mean", ends.mean())
