"""GPU tuning aid: per-CTA timeline of the persistent tcgen05 attention kernel
on a C2-shaped batch (T_q 256, 256 x 96-token items, H8 hd128).

Slots (clock64, relative to CTA start): 1+g = softmax saw S of block g,
32+g = P of block g handed to the MMA, 56+i = epilogue of item i done, 29 = end.
"""
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
trace = torch.zeros(256 * 64, dtype=torch.int64, device=dev)
for it in range(3):
    if it == 2:
        assert lib.sr_debug_attention_trace(C.c_void_p(trace.data_ptr())) == 0
    assert lib.sr_kernel_attention(C.c_void_p(qkv.data_ptr()),
                                   sp.ctypes.data_as(C.POINTER(C.c_int32)), M, H, hd,
                                   C.c_void_p(out.data_ptr()), None) == 0, lib.sr_last_error()
torch.cuda.synchronize()
lib.sr_debug_attention_trace(None)
t = trace.view(256, 64).cpu().numpy().astype(np.int64)
for b in [0, 1, 77, 147]:
    row = t[b]
    t0 = row[0]
    s = [int(row[1 + g] - t0) for g in range(24) if row[1 + g]]
    p = [int(row[32 + g] - t0) for g in range(24) if row[32 + g]]
    e = [int(row[56 + i] - t0) for i in range(8) if row[56 + i]]
    print(f"cta {b}: end {int(row[29] - t0)}")
    print("  S seen :", s)
    print("  P done :", p)
    print("  softmax per block:", [pp - ss for ss, pp in zip(s, p)])
    print("  wait for S:", [s[i + 1] - p[i] for i in range(min(len(s) - 1, len(p)))])
    print("  epilogues:", e)
ends = t[:148, 29] - t[:148, 0]
print("cta cycles: mean", ends.mean(), "min", ends.min(), "max", ends.max())
# per-CTA absolute start / end spread (the kernel ends with the slowest CTA)
starts = t[:148, 0]
endabs = t[:148, 29]
print("start spread (cycles)", int(starts.max() - starts.min()),
      "| end spread", int(endabs.max() - endabs.min()),
      "| longest CTA / mean", round(float(ends.max() / ends.mean()), 3))
