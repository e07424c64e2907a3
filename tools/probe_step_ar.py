"""Where the multi-GPU step's extra time goes: per-rank fused pass alone, pass + peer all-reduce, and the
all-reduce alone (R1, 10M tokens per rank, 150 chunks, 4 placements), CUDA events, max over ranks.
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/probe_step_ar.py"""
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
from paper_2508_09229_b200.shard import PeerSum  # noqa: E402

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
L, E, K, N, C = 58, 256, 8, 10_000_000, 150
m = mt.ModelSpec(L, E, K)
tr = mt.generate_trace(m, 1.2, N, C, rank)
rng = np.random.default_rng(0)
p = rng.integers(0, 7, (L, 32)).astype(np.uint8)
cost = mpl.CostMatrix(torch.as_tensor(p, device="cuda"))
pls = [mpl.Placement(rng.integers(0, 32, (L, E)).astype(np.int32)) for _ in range(4)]
tables, max_p = ev._group_tables(pls, [cost] * 4, m, 1)
bounds = _lib.to_dev(tr.chunk_bounds, torch.int64)
n = L * E + 4 * C
ps = PeerSum.create(n)
err = _lib.new_err()
sh = _lib.stream_handle()


def pass_(buf):
    _lib.call("mp_hist_score_ex_u8", _lib.ptr(tr.planes), tr.planes.shape[1], 0, N, L, K, E, _lib.ptr(bounds), C,
              _lib.ptr(tables), 1, max_p, _lib.ptr(buf[:L * E]), _lib.ptr(buf[L * E:]), _lib.ptr(err), 0, sh)


def step_a():
    pass_(ps.input())


def step_b():
    pass_(ps.input())
    ps.allreduce()


def step_c():
    ps.input()
    ps.allreduce()


def step_d():
    buf = ps.input()
    pass_(buf)
    dist.all_reduce(buf)


def timed(fn, reps):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / reps * 1e3], device="cuda")
    tmin = t.clone()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(tmin, op=dist.ReduceOp.MIN)
    return float(t.item()), float(tmin.item())


ta = timed(step_a, 100)
tb = timed(step_b, 100)
tc = timed(step_c, 400)
td = timed(step_d, 100)
ta2 = timed(step_a, 100)
tb2 = timed(step_b, 100)
ps.check()
if rank == 0:
    print(f"world {world}: pass alone {ta[0]:.1f} us (fastest rank {ta[1]:.1f}); pass + peer all-reduce {tb[0]:.1f} us; "
          f"pass + NCCL all_reduce {td[0]:.1f} us; all-reduce alone (back to back, incl. zeroing) {tc[0]:.1f} us; "
          f"again: pass alone {ta2[0]:.1f} / {ta2[1]:.1f}, pass + peer {tb2[0]:.1f}", flush=True)
dist.destroy_process_group()
