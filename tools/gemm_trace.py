"""GPU tuning aid: %globaltimer timeline of the CTA-pair GEMM on a C2 shape
(slots: 0 entry, 1 setup done, 2+i MMA of tile i issued, 24+i epilogue of
tile i done, 63 exit)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07309_b200._capi import lib  # noqa: E402

M = int(os.environ.get("GB_M", 24832))
dev = torch.device("cuda:0")
shapes = [("o0", 1024, 1024, 0), ("q0", 3072, 1024, 0), ("o2", 1024, 1024, 2)]
if os.environ.get("GT_SHAPES"):  # name:N:K:epi,...
    shapes = [(f[0], int(f[1]), int(f[2]), int(f[3]))
              for f in (x.split(":") for x in os.environ["GT_SHAPES"].split(","))]
trace = torch.zeros(256 * 64, dtype=torch.int64, device=dev)
for name, N, K, epi in shapes:
    A = (torch.randn(M, K, device=dev) * 0.5).bfloat16()
    B = (torch.randn(N, K, device=dev) * 0.05).bfloat16()
    Cm = torch.zeros(M, N, device=dev, dtype=torch.float32 if epi in (2, 3, 4) else torch.bfloat16)
    XB = torch.zeros(M, N, device=dev, dtype=torch.bfloat16)
    ST = torch.zeros(max(N, K) // 128, M, 2, device=dev)
    ST[..., 1] = 128.0
    CS = torch.randn(N, device=dev)
    st = torch.cuda.current_stream()
    for it in range(4):
        if it == 3:
            trace.zero_()
            assert lib.sr_debug_gemm_trace(C.c_void_p(trace.data_ptr())) == 0
        torch.cuda._sleep(2_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        if epi >= 4:
            rc = lib.sr_kernel_gemm_ln(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), M, N, K,
                                       C.c_void_p(Cm.data_ptr()), N, epi, C.c_void_p(XB.data_ptr()),
                                       C.c_void_p(ST.data_ptr()), K // 128, C.c_void_p(CS.data_ptr()),
                                       M, C.c_void_p(st.cuda_stream))
        else:
            rc = lib.sr_kernel_gemm(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), M, N, K,
                                    C.c_void_p(Cm.data_ptr()), N, epi, C.c_void_p(st.cuda_stream))
        assert rc == 0, lib.sr_last_error()
        b.record()
        torch.cuda.synchronize()
    lib.sr_debug_gemm_trace(None)
    ev_us = a.elapsed_time(b) * 1e3
    t = trace.view(256, 64).cpu().numpy()[:148].astype(np.int64)
    t = t[t[:, 0] > 0]  # CTAs that ran (a 4-CTA cluster grid uses 132)
    t0 = t[:, 0].min()
    rel = np.where(t > 0, t - t0, 0)
    entry, setup, exit_ = rel[:, 0], rel[:, 1], rel[:, 63]
    print(f"== {name} M{M} N{N} K{K} epi{epi}: event {ev_us:.1f} us, "
          f"trace span {(exit_.max()) / 1e3:.1f} us")
    print(f"  entry spread {entry.max() / 1e3:.2f} us; setup (entry->ready) median "
          f"{np.median(setup - entry) / 1e3:.2f} us max {(setup - entry).max() / 1e3:.2f}")
    print(f"  exit: min {exit_.min() / 1e3:.1f} median {np.median(exit_) / 1e3:.1f} max "
          f"{exit_.max() / 1e3:.1f} us")
    for cta in ([] if os.environ.get("GT_BRIEF") else [0, 2, 74, 146]):
        mma = [rel[cta, 2 + i] for i in range(22) if t[cta, 2 + i] > 0]
        epi_ = [rel[cta, 24 + i] for i in range(38) if t[cta, 24 + i] > 0]
        print(f"  cta {cta}: ready {rel[cta, 1] / 1e3:.2f} mma-done "
              f"{[round(x / 1e3, 2) for x in mma]} epi-done {[round(x / 1e3, 2) for x in epi_]} "
              f"exit {rel[cta, 63] / 1e3:.2f}")
    lead = t[0::2]
    d = np.diff(np.where(lead[:, 2:22] > 0, lead[:, 2:22], np.nan), axis=1)
    ep = []
    for c in range(0, t.shape[0], 2):
        for i in range(20):
            if t[c, 2 + i] > 0 and t[c, 24 + i] > 0:
                ep.append(t[c, 24 + i] - t[c, 2 + i])
    print(f"  per-tile MMA interval median {np.nanmedian(d) / 1e3:.2f} us (min "
          f"{np.nanmin(d) / 1e3:.2f}, max {np.nanmax(d) / 1e3:.2f}); epilogue (mma-done -> "
          f"epi-done) median {np.median(ep) / 1e3:.2f} us")
