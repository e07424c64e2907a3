"""torchrun check of the NCCL sharded path: every rank's all-reduced integers equal a one-GPU
run of the whole trace (rank 0 recomputes it).  Usage:
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/check_multigpu.py"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import moeplace.eval as ev  # noqa: E402
import moeplace.model_trace as mt  # noqa: E402
import moeplace.placement as mpl  # noqa: E402
import moeplace.topology as topo  # noqa: E402
from paper_2508_09229_b200.shard import sharded_evaluate  # noqa: E402

local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
m = mt.ModelSpec(58, 256, 8)
g = topo.build_topology(topo.TopologySpec("Dragonfly", 16, 4, 4))
d = topo.all_pairs_hops(g)
order = topo.locality_order(g, d)
attn = mt.default_attention_placement(m, order)
cost = mpl.cost_matrix(d, attn)
c = mpl.Constraints(64, 1)
pls = [mpl.place_round_robin(m, attn, order, c), mpl.place_greedy(m, attn, cost, c)]
N, C = 2_000_003, 150
freq, reps = sharded_evaluate(m, 1.2, N, C, 11, pls, cost)
# many placements over two topologies in one sharded evaluation (fused pass + gather passes)
g2 = topo.build_topology(topo.TopologySpec("FatTree", 16, 4, 4))
d2 = topo.all_pairs_hops(g2)
cost2 = mpl.cost_matrix(d2, mt.default_attention_placement(m, topo.locality_order(g2, d2)))
rng = np.random.default_rng(0)
many = [mpl.Placement(np.stack([rng.permutation(256) for _ in range(58)])) for _ in range(21)]
mcost = [cost if i % 2 else cost2 for i in range(21)]
_, many_reps = sharded_evaluate(m, 1.2, N, C, 11, many, mcost)
sig = torch.tensor([int(freq.counts.sum()), sum(r.hop_sum for r in reps)], dtype=torch.int64, device="cuda")
allsig = [torch.zeros_like(sig) for _ in range(world)]
dist.all_gather(allsig, sig)
if rank == 0:
    tr = mt.generate_trace(m, 1.2, N, C, 11)
    f1, r1 = ev.evaluate_with_stats(tr, pls, cost)
    assert np.array_equal(f1.counts, freq.counts), "counts differ"
    assert [r.chunk_hop_sums for r in r1] == [r.chunk_hop_sums for r in reps], "hop sums differ"
    assert all(torch.equal(s, allsig[0]) for s in allsig), "ranks disagree"
    want_many = ev.score_sums(tr, many, mcost)
    assert [r.chunk_hop_sums for r in many_reps] == want_many.tolist(), "many-placement sums differ"
    print(f"multigpu ok: world={world} counts and per-chunk hop sums bit-identical to 1 GPU; "
          f"RR {reps[0].mean_hops_per_token:.4f} greedy {reps[1].mean_hops_per_token:.4f}")
dist.barrier()
dist.destroy_process_group()
