"""Probe (not product code): does the fused count-contract kernel slow down after torch.distributed / NCCL
initialisation or a symmetric-memory allocation in the same process?  Times mp_hist_score_ex_u8 (R1, 10M
tokens, 150 chunks, 4 placements) before and after each step.  Run under torchrun (any world size)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import moeplace.eval as ev  # noqa: E402
import moeplace.model_trace as mt  # noqa: E402
import moeplace.placement as mpl  # noqa: E402
from paper_2508_09229_b200 import _lib  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
L, E, K, N, C = 58, 256, 8, 10_000_000, 150
m = mt.ModelSpec(L, E, K)
tr = mt.generate_trace(m, 1.2, N, C, 0)
rng = np.random.default_rng(0)
p = rng.integers(0, 7, (L, 32)).astype(np.uint8)
cost = mpl.CostMatrix(torch.as_tensor(p, device="cuda"))
pls = [mpl.Placement(rng.integers(0, 32, (L, E)).astype(np.int32)) for _ in range(4)]
tables, max_p = ev._group_tables(pls, [cost] * 4, m, 1)
bounds = _lib.to_dev(tr.chunk_bounds, torch.int64)
err = _lib.new_err()


def run(counts, sums):
    _lib.call("mp_hist_score_ex_u8", _lib.ptr(tr.planes), tr.planes.shape[1], 0, N, L, K, E, _lib.ptr(bounds), C,
              _lib.ptr(tables), 1, max_p, _lib.ptr(counts), _lib.ptr(sums), _lib.ptr(err), 0, _lib.stream_handle())


def timed(counts, sums, reps=20):
    for _ in range(3):
        run(counts, sums)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        run(counts, sums)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


cnt = torch.zeros(L * E, dtype=torch.int64, device="cuda")
sums = torch.zeros(4 * C, dtype=torch.int64, device="cuda")
out = {"plain": timed(cnt, sums)}
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
out["after_nccl_init"] = timed(cnt, sums)
x = torch.ones(1024, device="cuda")
dist.all_reduce(x)
torch.cuda.synchronize()
out["after_first_all_reduce"] = timed(cnt, sums)
from paper_2508_09229_b200.shard import PeerSum  # noqa: E402
ps = PeerSum.create(L * E + 4 * C)
out["after_symm_alloc"] = timed(cnt, sums)
buf = ps.input()
out["outputs_in_symm_memory"] = timed(buf[:L * E], buf[L * E:])
out["plain_again"] = timed(cnt, sums)
print(dist.get_rank(), {k: round(v, 1) for k, v in out.items()}, flush=True)
dist.destroy_process_group()
