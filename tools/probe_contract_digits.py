"""Probe (not product code): does the tcgen05 contraction's time scale with the digit operand (B rows =
C x digits, re-read from L2 by every pe-tile CTA of a k-range) or with the pe operand?  Config-4
shape (P = 4096 x L*E = 14848, C = 150) with 1 / 2 / 3 count digits, and P = 1024 / 2048 / 4096."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_09229_b200 import _lib  # noqa: E402
if len(sys.argv) > 1:  # an experiment build of the library
    from pathlib import Path
    _lib.LIB_PATH = Path(sys.argv[1])
from paper_2508_09229_b200 import eval as ev  # noqa: E402

LE, C = 58 * 256, 150
g = torch.Generator(device="cuda").manual_seed(0)


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


res = {}
for P in (1024, 2048, 4096):
    pe = torch.randint(0, 13, (P, LE), dtype=torch.uint8, device="cuda", generator=g)
    for ndig, mx in ((1, 255), (2, 6666), (3, 70000)):
        cnt = torch.randint(0, mx + 1, (C, LE), dtype=torch.int64, device="cuda", generator=g)
        d = ev.CountDigits(cnt, mx)
        out = torch.zeros((P, C), dtype=torch.int64, device="cuda")
        res[f"P{P}_digits{ndig}_ms"] = timeit(lambda: d.contract(pe, out))
print(json.dumps(res, indent=1))
