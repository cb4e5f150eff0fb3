"""GPU tuning aid: per-launch time of the pair GEMM when launched back to back
(1, 2, 5, 10 launches between one event pair), against a single launch after
a sleep kernel, and the same through a captured CUDA graph."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07309_b200._capi import lib  # noqa: E402

M = 24832
dev = torch.device("cuda:0")
for name, N, K, epi in [("q0", 3072, 1024, 0), ("o2", 1024, 1024, 2), ("o0", 1024, 1024, 0)]:
    A = (torch.randn(M, K, device=dev) * 0.5).bfloat16()
    B = (torch.randn(N, K, device=dev) * 0.05).bfloat16()
    Cm = torch.zeros(M, N, device=dev, dtype=torch.float32 if epi in (2, 3) else torch.bfloat16)
    st = torch.cuda.current_stream()

    def launch():
        rc = lib.sr_kernel_gemm(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), M, N, K,
                                C.c_void_p(Cm.data_ptr()), N, epi, C.c_void_p(st.cuda_stream))
        assert rc == 0, lib.sr_last_error()

    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    res = {}
    for n in (1, 2, 5, 10):
        ts = []
        for rep in range(5):
            torch.cuda._sleep(3_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(n):
                launch()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / n)
        res[n] = sorted(ts)[2]
    # graph of 10 launches
    g = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        st = s2
        with torch.cuda.graph(g, stream=s2):
            for _ in range(10):
                launch()
    st = torch.cuda.current_stream()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for rep in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / 10)
    print(name, {k: round(v, 1) for k, v in res.items()}, "graph10", round(sorted(ts)[2], 1), "us/launch",
          flush=True)
