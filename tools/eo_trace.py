"""GPU tuning aid: clock64 timeline of the block-parity attention kernel
(attention_eo.cu, SRK_ATTN=eo; slots documented there) on a C2-shaped layer."""
import ctypes as C
import os
import sys

import numpy as np
import torch

os.environ["SRK_ATTN"] = "eo"
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
trace = torch.zeros(148 * 256, dtype=torch.int64, device=dev)
for it in range(3):
    if it == 2:
        assert lib.sr_debug_attention_trace(C.c_void_p(trace.data_ptr())) == 0
    assert lib.sr_kernel_attention(C.c_void_p(qkv.data_ptr()),
                                   sp.ctypes.data_as(C.POINTER(C.c_int32)), M, H, hd,
                                   C.c_void_p(out.data_ptr()), None) == 0, lib.sr_last_error()
torch.cuda.synchronize()
lib.sr_debug_attention_trace(None)
t = trace.view(148, 256).cpu().numpy().astype(np.int64)
tot = t[:, 225] - t[:, 224]
print("cycles per CTA: mean", int(tot.mean()), "min", int(tot.min()), "max", int(tot.max()))
for b in [0, 77]:
    r = t[b]
    t0 = r[224]
    rel = lambda v: int(v - t0) if v else -1
    print(f"--- CTA {b}")
    for x in range(2):
        print(f"slot {x} (S seen, P handed, dur):",
              " ".join(f"({rel(r[2 * (24 * x + k)])},{rel(r[2 * (24 * x + k) + 1])},{int(r[2 * (24 * x + k) + 1] - r[2 * (24 * x + k)])})" for k in range(12)))
    print("MMA g: (PV waits done, next S issued):",
          " ".join(f"{g}:({rel(r[96 + 2 * g])},{rel(r[97 + 2 * g])})" for g in range(24)))
