"""ncu target (not product code): the config-4 contraction alone, a few launches
(`ncu --set full -k regex:contract_tc -c 2 python tools/prof_contract.py`)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_09229_b200 import eval as ev  # noqa: E402

P, LE, C = 4096, 58 * 256, 150
ctas = int(sys.argv[1]) if len(sys.argv) > 1 else 0
g = torch.Generator(device="cuda").manual_seed(0)
pe = torch.randint(0, 13, (P, LE), dtype=torch.uint8, device="cuda", generator=g)
cnt = torch.randint(0, 6667, (C, LE), dtype=torch.int64, device="cuda", generator=g)
d = ev.CountDigits(cnt, 6666)
out = torch.zeros((P, C), dtype=torch.int64, device="cuda")
for _ in range(3):
    d.contract(pe, out, ctas=ctas)
torch.cuda.synchronize()
print("ok")
