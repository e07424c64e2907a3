"""Probe (not product code): one config-4 contraction launch with an instrumented build (MP_TC_PROFILE) -- prints per-warp phase times."""
import os, sys
sys.path.insert(0, '/root/repo')
from pathlib import Path
from paper_2508_09229_b200 import _lib
_lib.LIB_PATH = Path(sys.argv[1])
import torch
from paper_2508_09229_b200 import eval as ev
LE, C, P = 58 * 256, 150, 4096
g = torch.Generator(device="cuda").manual_seed(0)
pe = torch.randint(0, 13, (P, LE), dtype=torch.uint8, device="cuda", generator=g)
cnt = torch.randint(0, 6667, (C, LE), dtype=torch.int64, device="cuda", generator=g)
d = ev.CountDigits(cnt, 6666)
out = torch.zeros((P, C), dtype=torch.int64, device="cuda")
for _ in range(3):
    d.contract(pe, out)
torch.cuda.synchronize()
