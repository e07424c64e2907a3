"""Times the packed-vector sum (R1 config 2: 58*256 + 4*150 int64) with the library's peer-memory
kernel (shard.PeerSum: NVLS multimem.ld_reduce / P2P) against torch.distributed.all_reduce (NCCL),
CUDA events, max over ranks, and checks both give the same integers.
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/time_allreduce.py"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_09229_b200.shard import PeerSum  # noqa: E402

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
n = 58 * 256 + 4 * 150
ps = PeerSum.create(n)
g = torch.Generator(device="cuda").manual_seed(rank)
src = torch.randint(0, 1 << 40, (n,), dtype=torch.int64, device="cuda", generator=g)
ref = src.clone()
dist.all_reduce(ref)
ps.input().copy_(src)
res = ps.allreduce()
torch.cuda.synchronize()
ps.check()
ok = torch.equal(res, ref)


def timed(fn, reps=200):
    for _ in range(10):
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
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


x = src.clone()
t_peer = timed(lambda: (ps.input(), ps.allreduce()))
t_nccl = timed(lambda: dist.all_reduce(x))
ps.check()
if rank == 0:
    print(f"world {world}: n = {n} int64; peer-memory sum (multicast={'yes' if ps.mcs[0] else 'no'}) {t_peer:.1f} us, "
          f"NCCL all_reduce {t_nccl:.1f} us; bit-identical: {ok}", flush=True)
dist.destroy_process_group()
