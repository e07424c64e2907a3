"""Probe (not product code): the factorized contraction at BASELINE config 4 (P = 4096 pe rows x
L*E = 14848, C = 150 chunks of ~6.7k tokens, 2 count digits).  Times the product path
(``mp_count_digits_u8`` + ``mp_contract_tc_u8``, tcgen05 kind::i8) per split-K factor against the
CUDA-core int64 kernel and, for context only, cuBLASLt's int8 GEMM of the same operand sizes
(torch._int_mm -- not on any product path)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_09229_b200 import _lib  # noqa: E402
from paper_2508_09229_b200 import eval as ev  # noqa: E402

P, LE, C = 4096, 58 * 256, 150
g = torch.Generator(device="cuda").manual_seed(0)
pe = torch.randint(0, 13, (P, LE), dtype=torch.uint8, device="cuda", generator=g)
cnt = torch.randint(0, 6667, (C, LE), dtype=torch.int64, device="cuda", generator=g)


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
d = ev.CountDigits(cnt, 6666)
out = torch.zeros((P, C), dtype=torch.int64, device="cuda")
ref = torch.zeros((P, C), dtype=torch.int64, device="cuda")
_lib.call("mp_contract_counts", _lib.ptr(cnt), C, _lib.ptr(pe), P, LE, _lib.ptr(ref), _lib.stream_handle())
res["CountDigits_python_call_ms"] = timeit(lambda: ev.CountDigits(cnt, 6666))
res["count_digits_u8_kernel_ms"] = timeit(lambda: _lib.call("mp_count_digits_u8", _lib.ptr(cnt), C, LE, 2, d.ldd,
                                                            _lib.ptr(d.buf), _lib.ptr(d.err), _lib.stream_handle()))
for sp in (0, 64, 128, 148, 296, -32, -64, -74):
    out.zero_()
    d.contract(pe, out, ctas=sp)
    ok = torch.equal(out, ref)
    res[f"contract_tc_ctas{sp}_ms"] = timeit(lambda: d.contract(pe, out, ctas=sp))
    res[f"contract_tc_ctas{sp}_exact"] = bool(ok)
res["contract_tc_total_ms"] = timeit(lambda: ev.contract_tc(cnt, pe, max_count=6666))
res["cuda_core_int64_ms"] = timeit(lambda: _lib.call("mp_contract_counts", _lib.ptr(cnt), C, _lib.ptr(pe), P, LE,
                                                     _lib.ptr(out), _lib.stream_handle()), reps=5)
B = torch.zeros((304, LE), dtype=torch.int8, device="cuda")
res["cublaslt_int8_4096x304x14848_ms_context_only"] = timeit(lambda: torch._int_mm(pe.view(torch.int8), B.t()))
flops = 2 * P * 304 * LE
best = min(v for k, v in res.items() if k.startswith("contract_tc_ctas") and k.endswith("_ms"))
res["tensor_tops_best"] = flops / (best / 1e3) / 1e12
res["pe_read_GBps_best"] = P * LE / (best / 1e3) / 1e9
print(json.dumps(res, indent=1))
