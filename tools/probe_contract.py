"""Probe (not product code): where the factorized contraction's time goes at config 4
(P = 4096 pe rows x L*E = 14848, C = 150 chunks of ~6.7k tokens).  Times the current
``eval.contract_tc`` and its parts, and a one-GEMM variant with the count digits stacked
along N."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_09229_b200 import eval as ev  # noqa: E402

P, LE, C = 4096, 58 * 256, 150
g = torch.Generator(device="cuda").manual_seed(0)
pe = torch.randint(0, 13, (P, LE), dtype=torch.uint8, device="cuda", generator=g)
cnt = torch.randint(0, 6667, (C, LE), dtype=torch.int64, device="cuda", generator=g)


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


ref = ev.contract_tc(cnt, pe)
print(f"contract_tc                    {timeit(lambda: ev.contract_tc(cnt, pe)):.4f} ms")
Cp = 152
B = torch.zeros((2 * Cp, LE), dtype=torch.int8, device="cuda")


def stacked():
    B[:C].copy_((cnt & 127).to(torch.int8))
    B[Cp:Cp + C].copy_(((cnt >> 7) & 127).to(torch.int8))
    r = torch._int_mm(pe.view(torch.int8), B.t())
    return r[:, :C].to(torch.int64) + (r[:, Cp:Cp + C].to(torch.int64) << 7)


assert torch.equal(stacked(), ref)
print(f"stacked digits, one GEMM       {timeit(stacked):.4f} ms")
print(f"  digit split (2 planes)       {timeit(lambda: (B[:C].copy_((cnt & 127).to(torch.int8)), B[Cp:Cp + C].copy_(((cnt >> 7) & 127).to(torch.int8)))):.4f} ms")
print(f"  _int_mm {P}x{2 * Cp}x{LE}    {timeit(lambda: torch._int_mm(pe.view(torch.int8), B.t())):.4f} ms")
r = torch._int_mm(pe.view(torch.int8), B.t())
print(f"  combine                      {timeit(lambda: r[:, :C].to(torch.int64) + (r[:, Cp:Cp + C].to(torch.int64) << 7)):.4f} ms")
Bt = B.t().contiguous()
for n in (152, 304):
    Bn = torch.zeros((n, LE), dtype=torch.int8, device="cuda")
    print(f"  _int_mm {P}x{n}x{LE}           {timeit(lambda: torch._int_mm(pe.view(torch.int8), Bn.t())):.4f} ms")
# transpose roles: counts as the M operand (rows = chunks' digits), pe^T as N
print(f"  _int_mm {2 * Cp}x{P}x{LE} (swapped) {timeit(lambda: torch._int_mm(B, pe.view(torch.int8).t())):.4f} ms")
