"""Host->device copy rates on the box: pageable vs pinned, and host memcpy."""
import time

import numpy as np
import torch

n = 33_554_432
src = np.random.default_rng(0).standard_normal(n // 4).astype(np.float32)
dev = torch.empty(n // 4, dtype=torch.float32, device="cuda")
pin = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
t_src = torch.from_numpy(src)


def rate(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return n * reps / (time.perf_counter() - t) / 1e9


print("pageable->dev GB/s", round(rate(lambda: dev.copy_(t_src)), 1))
print("pinned->dev GB/s", round(rate(lambda: dev.copy_(pin, non_blocking=True)), 1))
print("host memcpy (1 thread) GB/s", round(rate(lambda: pin.copy_(t_src)), 1))
dst = np.empty_like(src)
print("numpy copy GB/s", round(rate(lambda: np.copyto(dst, src)), 1))
