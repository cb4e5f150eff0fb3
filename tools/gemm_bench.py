"""GPU tuning aid: our tcgen05 GEMMs vs cuBLAS (torch.matmul) on the C2 layer
shapes (M = 24,832 packed rows, d 1024, ff 1536). Kernel time only: a
torch.cuda._sleep ahead of each call hides the host-side tensor-map setup of
sr_kernel_gemm from the CUDA events."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_07309_b200._capi import lib  # noqa: E402

M = int(os.environ.get("GB_M", 24832))
SHAPES = [("qkv", 3072, 1024, 0), ("o", 1024, 1024, 2), ("w_in", 1536, 1024, 1),
          ("w_out", 1024, 1536, 2),
          # folded-LN epilogues (4 residual + statistics, 5 LN-projection, 6 + GELU)
          ("qkv_ln", 3072, 1024, 5), ("o_ln", 1024, 1024, 4), ("w_in_ln", 1536, 1024, 6),
          ("wout_ln", 1024, 1536, 4)]
if os.environ.get("GB_SHAPES"):  # name:N:K:epi,...
    SHAPES = [(f[0], int(f[1]), int(f[2]), int(f[3]))
              for f in (x.split(":") for x in os.environ["GB_SHAPES"].split(","))]
dev = torch.device("cuda:0")
torch.manual_seed(0)


FLUSH = torch.empty(0)
if os.environ.get("GB_FLUSH"):  # cold L2 before every timed call
    FLUSH = torch.empty(64 << 20, dtype=torch.float32, device=dev)


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        if FLUSH.numel():
            FLUSH.fill_(1.0)
        torch.cuda._sleep(2_000_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


for name, N, K, epi in SHAPES:
    A = (torch.randn(M, K, device=dev) * 0.5).bfloat16()
    B = (torch.randn(N, K, device=dev) * 0.05).bfloat16()
    if epi in (2, 3, 4):
        Cm = torch.zeros(M, N, device=dev, dtype=torch.float32)
    else:
        Cm = torch.zeros(M, N, device=dev, dtype=torch.bfloat16)
    XB = torch.zeros(M, N, device=dev, dtype=torch.bfloat16)
    P = K // 128
    ST = torch.zeros(max(N, K) // 128, M, 2, device=dev)
    ST[..., 1] = 128.0  # unit variance partials
    CS = torch.randn(N, device=dev)

    def ours():
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        if epi >= 4:
            rc = lib.sr_kernel_gemm_ln(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), M, N, K,
                                       C.c_void_p(Cm.data_ptr()), N, epi, C.c_void_p(XB.data_ptr()),
                                       C.c_void_p(ST.data_ptr()), P, C.c_void_p(CS.data_ptr()), M, s)
        else:
            rc = lib.sr_kernel_gemm(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), M, N, K,
                                    C.c_void_p(Cm.data_ptr()), N, epi, s)
        assert rc == 0, lib.sr_last_error()

    def cublas():
        torch.matmul(A, B.t())

    ours()
    cublas()
    t_o, t_c = timed(ours), timed(cublas)
    fl = 2.0 * M * N * K
    print(f"{name:6s} M{M} N{N} K{K} epi{epi}: ours {t_o * 1e3:7.1f} us {fl / t_o / 1e9:7.0f} TF/s"
          f" | cuBLAS {t_c * 1e3:7.1f} us {fl / t_c / 1e9:7.0f} TF/s", flush=True)
