"""GPU tuning aid: the residual GEMM with the next LayerNorm overlapped
(epilogue 7 + layer_norm_after on a side stream, sr_kernel_gemm_resid_ln) on
a C2 shape: time vs the plain residual GEMM, parity of the LN output."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07309_b200._capi import lib  # noqa: E402

M, N, K = 24832, 1024, int(os.environ.get("K", 1024))
dev = torch.device("cuda:0")
A = (torch.randn(M, K, device=dev) * 0.5).bfloat16()
B = (torch.randn(N, K, device=dev) * 0.05).bfloat16()
X = torch.randn(M, N, device=dev)
G = torch.rand(N, device=dev) + 0.5
O = torch.zeros(M, N, device=dev, dtype=torch.bfloat16)
cnt = torch.zeros(M // 128 + 8, device=dev, dtype=torch.int32)
trace = torch.zeros(256 * 64, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream().cuda_stream
vp = lambda t: C.c_void_p(t.data_ptr())
for mode in ("resid", "resid_ln"):
    for it in range(4):
        if it == 3 and mode == "resid_ln":
            trace.zero_()
            assert lib.sr_debug_gemm_trace(vp(trace)) == 0
        torch.cuda._sleep(2_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if mode == "resid":
            rc = lib.sr_kernel_gemm(vp(A), vp(B), M, N, K, vp(X), N, 2, C.c_void_p(st))
        else:
            rc = lib.sr_kernel_gemm_resid_ln(vp(A), vp(B), M, N, K, vp(X), vp(G), vp(O), vp(cnt),
                                             C.c_void_p(st))
        assert rc == 0, lib.sr_last_error()
        b.record()
        torch.cuda.synchronize()
    print(f"{mode}: {a.elapsed_time(b) * 1e3:.1f} us")
lib.sr_debug_gemm_trace(None)
# parity of the overlapped LayerNorm against torch on the same x
ref = torch.nn.functional.layer_norm(X, (N,), eps=1e-5) * G
err = (O.float() - ref).abs().max().item()
print(f"max |LN-after - torch| = {err:.3e}; counters back to zero: {int(cnt.abs().sum().item()) == 0}")
