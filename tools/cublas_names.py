"""Prints the cuBLAS kernel names (tile / cluster shapes) for the C2 GEMM shapes."""
import torch
from torch.profiler import profile, ProfilerActivity
M = 24832
dev = torch.device("cuda:0")
for N, K in [(3072, 1024), (1024, 1024), (1536, 1024), (1024, 1536)]:
    A = torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(N, K, device=dev).bfloat16()
    torch.matmul(A, B.t())
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
        torch.matmul(A, B.t())
        torch.cuda.synchronize()
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            print(N, K, e.name[:300])
