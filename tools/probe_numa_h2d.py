"""Probe (not product code): concurrent pinned host->device bandwidth of N ranks, with and without
binding each rank (and its pinned buffer's first touch) to the CPUs local to its GPU.
  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/probe_numa_h2d.py"""
import os
import time

import torch
import torch.distributed as dist

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
props = torch.cuda.get_device_properties(local)
bus = f"{getattr(props, 'pci_domain_id', 0):04x}:{getattr(props, 'pci_bus_id', 0):02x}:{getattr(props, 'pci_device_id', 0):02x}.0"


def sysfs(name):
    try:
        return open(f"/sys/bus/pci/devices/{bus}/{name}").read().strip()
    except OSError as e:
        return f"? ({e.__class__.__name__})"


numa, cpus = sysfs("numa_node"), sysfs("local_cpulist")
print(f"rank {rank}: gpu {local} pci {bus} numa {numa} cpus {cpus} affinity {len(os.sched_getaffinity(0))}", flush=True)
NB = 4 << 30


def run(tag):
    h = torch.empty(NB, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(NB, dtype=torch.uint8, device="cuda")
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    dist.barrier()
    t = torch.tensor([dt])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"{tag}: {world} ranks x 4 GiB concurrently in {t.item() * 1e3:.1f} ms -> aggregate "
              f"{world * NB / t.item() / 1e9:.1f} GB/s", flush=True)
    del h, d


run("default affinity")


def parse(cl):
    out = set()
    for part in cl.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.update(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


try:
    os.sched_setaffinity(0, parse(cpus))
    run("bound to the GPU's local CPUs")
except Exception as e:  # noqa: BLE001
    if rank == 0:
        print("binding failed:", e)
dist.destroy_process_group()
