"""Raw pinned host -> device bandwidth (the e2e path's ceiling)."""
import time

import torch

for gb in (1, 4):
    n = gb << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"H2D {gb} GiB: {ms:.1f} ms  {n / ms / 1e6:.1f} GB/s")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    half = n // 2
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        with torch.cuda.stream(s1):
            d[:half].copy_(h[:half], non_blocking=True)
        with torch.cuda.stream(s2):
            d[half:].copy_(h[half:], non_blocking=True)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / 3 * 1e3
    print(f"H2D {gb} GiB on 2 streams: {ms:.1f} ms  {n / ms / 1e6:.1f} GB/s")
