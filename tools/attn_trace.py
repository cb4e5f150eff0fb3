"""GPU tuning aid: per-CTA timeline of the tcgen05 attention kernel on a C2-shaped batch."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07309_b200._capi import lib
H, hd, tq, L, n = 8, 128, 256, 96, 256
spans = [[0, 0, 0, 0]] * tq
cur = tq
for _ in range(n):
    spans += [[0, tq, cur, 0]] * L
    cur += L
M = len(spans); d = H * hd
dev = torch.device("cuda:0")
qkv = (torch.randn(M, 3 * d, device=dev) * 0.5).bfloat16()
out = torch.zeros(M, d, dtype=torch.bfloat16, device=dev)
sp = np.asarray(spans, np.int32).reshape(-1)
trace = torch.zeros(256 * 64, dtype=torch.int64, device=dev)
for it in range(3):
    if it == 2:
        assert lib.sr_debug_attention_trace(C.c_void_p(trace.data_ptr())) == 0
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    assert lib.sr_kernel_attention(C.c_void_p(qkv.data_ptr()), sp.ctypes.data_as(C.POINTER(C.c_int32)), M, H, hd, C.c_void_p(out.data_ptr()), None) == 0, lib.sr_last_error()
    e.record(); torch.cuda.synchronize()
    print("iter", it, "ms", s.elapsed_time(e))
lib.sr_debug_attention_trace(None)
t = trace.view(256, 64).cpu().numpy()
names = {0: "start", 1: "setup", 2: "q_full", 27: "epi", 29: "end"}
for b in [0, 1, 2, 3, 10, 50, 100, 150, 200, 255]:
    row = t[b]; t0 = row[0]
    ev = [(k, int(row[k] - t0)) for k in range(30) if row[k] != 0]
    nb = int(row[30])
    parts = []
    for k, v in ev:
        lab = names.get(k) or (f"PV{k-3}" if 3 <= k < 11 else f"S{k-11}" if 11 <= k < 19 else f"P{k-19}")
        parts.append(f"{lab}:{v}")
    print(f"cta {b:3d} sm {int(row[31]):3d} nblk {nb}: " + " ".join(parts))
ends = t[:, 29] - t[:, 0]
print("cta cycles: mean", ends[ends > 0].mean(), "min", ends[ends > 0].min(), "max", ends.max())
