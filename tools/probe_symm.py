"""Probe (not product code): torch symmetric memory on this box -- peer pointers, signal pads and
multicast support for a peer-memory reduction of the packed result vector.
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/probe_symm.py"""
import os
import time

import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
group = dist.group.WORLD
symm.enable_symm_mem_for_group(group.group_name)
n = 24_600
buf = symm.empty(n, dtype=torch.int64, device="cuda")
buf.fill_(rank + 1)
hdl = symm.rendezvous(buf, group.group_name)
out = {"rank": rank, "world": world, "buffer_ptrs": [hex(p) for p in hdl.buffer_ptrs],
       "signal_pad_ptrs": [hex(p) for p in hdl.signal_pad_ptrs], "multicast_ptr": hex(hdl.multicast_ptr),
       "signal_pad_size": symm.get_signal_pad_size()}
hdl.barrier()
peer = hdl.get_buffer((rank + 1) % world, (n,), torch.int64)
out["peer_first"] = int(peer[0].item())
# NCCL all_reduce of the same vector for reference timing
x = torch.ones(n, dtype=torch.int64, device="cuda")
for _ in range(5):
    dist.all_reduce(x)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(50):
    dist.all_reduce(x)
ev[1].record()
torch.cuda.synchronize()
out["nccl_allreduce_us"] = ev[0].elapsed_time(ev[1]) / 50 * 1e3
print(out, flush=True)
dist.destroy_process_group()
