"""GPU tuning aid: device time of one segment-masked attention launch on a
C2-shaped layer (T_q 256, 256 x 96-token items, H8 hd128), CUDA events over
20 back-to-back launches after warm-up, plus the max |diff| against a
reference output file (same inputs, seed 0) when given. The kernel variant
follows the SRK_ATTN* environment (one process per variant)."""
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
g = torch.Generator(device=dev).manual_seed(0)
qkv = (torch.randn(M, 3 * d, device=dev, generator=g) * 0.5).bfloat16()
out = torch.zeros(M, d, dtype=torch.bfloat16, device=dev)
sp = np.asarray(spans, np.int32).reshape(-1)


def run():
    assert lib.sr_kernel_attention(C.c_void_p(qkv.data_ptr()), sp.ctypes.data_as(C.POINTER(C.c_int32)),
                                   M, H, hd, C.c_void_p(out.data_ptr()), None) == 0, lib.sr_last_error()


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / reps * 1000
tag = os.environ.get("TAG", "attn")
if os.environ.get("SAVE_OUT"):
    np.save(f"/tmp/{tag}_out.npy", out.float().cpu().numpy())
ref = sys.argv[1] if len(sys.argv) > 1 else None
diff = None
if ref and os.path.exists(ref):
    diff = float(np.abs(np.load(ref) - out.float().cpu().numpy()).max())
print(f"{tag}: {us:.1f} us per launch (incl. launch gaps), max|diff| vs ref {diff}")
