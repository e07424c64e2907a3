"""Probe (not product code): file-write strategies for the device text writer (2.1 GB of text from
a 1M-token R1 trace): the pinned ring with parallel pwrite, the same after posix_fallocate, and a
single buffered write, each into a fresh file."""
import os
import sys
import tempfile
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import moeplace.model_trace as mt  # noqa: E402
from paper_2508_09229_b200 import model_trace as pmt  # noqa: E402

n = 2_100_000_000
src = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
d = tempfile.mkdtemp()
print("tmp fs:", os.statvfs(d).f_bsize, d)


def run(name, fn):
    p = os.path.join(d, name)
    if os.path.exists(p):
        os.remove(p)
    torch.cuda.synchronize()
    a = time.perf_counter()
    fn(p)
    dt = time.perf_counter() - a
    print(f"{name:28s} {dt:6.3f} s  {n / dt / 1e9:6.2f} GB/s")
    os.remove(p)


def ring(p):
    with open(p, "wb") as f:
        pmt._device_to_file(src, n, f.fileno(), 0)


def ring_falloc(p):
    with open(p, "wb") as f:
        os.posix_fallocate(f.fileno(), 0, n)
        pmt._device_to_file(src, n, f.fileno(), 0)


def single(p):
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h.copy_(src)
    with open(p, "wb") as f:
        f.write(memoryview(h.numpy()))


def ring_trunc(p):
    with open(p, "wb") as f:
        os.ftruncate(f.fileno(), n)
        pmt._device_to_file(src, n, f.fileno(), 0)


for _ in range(2):
    for nm, fn in [("ring", ring), ("ring+fallocate", ring_falloc), ("ring+ftruncate", ring_trunc),
                   ("single pinned write", single)]:
        run(nm, fn)
print("d2h only", end=" ")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
torch.cuda.synchronize()
a = time.perf_counter()
h.copy_(src)
print(f"{time.perf_counter() - a:.3f} s")
