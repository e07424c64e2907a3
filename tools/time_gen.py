"""Times the trace generator kernel (mp_gen_trace) for R1 (L=58, E=256, K=8) traces with CUDA events.
  python tools/time_gen.py [--tokens N] [--s zipf] [--lib path]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import moeplace.model_trace as mt  # noqa: E402
from paper_2508_09229_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=10_000_000)
ap.add_argument("--s", type=float, default=1.2)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--lib")
a = ap.parse_args()
if a.lib:
    from pathlib import Path
    _lib.LIB_PATH = Path(a.lib)
m = mt.ModelSpec(58, 256, 8)
for s in (a.s, 0.0, 2.0):
    tr = mt.generate_trace(m, s, a.tokens, 150, 0)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(a.reps):
        mt.generate_trace(m, s, a.tokens, 150, 0)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / a.reps
    gb = a.tokens * 58 * 8 / 1e9
    print(f"zipf {s}: generate_trace {a.tokens} R1 tokens {ms:.2f} ms  ({gb / ms * 1e3:.1f} GB/s written)")
