"""Pinned host<->device copy bandwidth on this box (diagnostics)."""
import time
import torch

for mb in (1, 4, 16, 64, 256):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(reps):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{mb:4d} MB  H2D {reps * n / (t1 - t0) / 1e9:6.1f} GB/s  D2H {reps * n / (t2 - t1) / 1e9:6.1f} GB/s")
