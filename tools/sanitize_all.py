"""Exercises every device entry point on small, awkward inputs (ragged N, unaligned views,
K != 8, empty chunks, host streaming, parser/writer) — for compute-sanitizer runs:
  compute-sanitizer --tool memcheck python tools/sanitize_all.py"""
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import moeplace.eval as ev  # noqa: E402
import moeplace.model_trace as mt  # noqa: E402
import moeplace.placement as mpl  # noqa: E402
import moeplace.search as se  # noqa: E402
import moeplace.solver as sv  # noqa: E402
import moeplace.topology as topo  # noqa: E402

mt.STREAM_BLOCK_TOKENS = 333
for (L, E, K) in [(3, 64, 8), (2, 16, 5), (4, 256, 1)]:
    m = mt.ModelSpec(L, E, K)
    g = topo.build_topology(topo.TopologySpec("DragonflySparse", 5, 2, 2))
    d = topo.all_pairs_hops(g)
    _ = d.dist
    order = topo.locality_order(g, d)
    attn = mt.default_attention_placement(m, order)
    cost = mpl.cost_matrix(d, attn)
    c = mpl.Constraints(64, 8)
    tr = mt.generate_trace(m, 1.2, 1001, 17, 3)
    rng = np.random.default_rng(0)
    pls = [mpl.Placement(rng.integers(0, g.n_devices, (L, E))) for _ in range(18)]
    for v in (tr, tr.view(3, 11), tr.view(16, 17)):
        mt.estimate_frequencies(v, m)
        ev.score_sums(v, pls, cost)
        ev.evaluate_with_stats(v, pls[:4], cost)
        ev.score_sums_factorized(v, pls, cost)
        ev.score_sums_factorized(v, pls[:3], cost, contraction="cuda")
        ev.token_hops_all(v, pls[:5], cost)
        ev.evaluate_dedup(v, pls[:5], cost)
        ev.communication_map(v, pls[0], cost)
    host = tr.to_host(pin=True)
    ev.score_sums(host, pls[:6], cost)
    ev.evaluate_with_stats(host, pls[:4], cost)
    inst = sv.build_instance(cost, mt.estimate_frequencies(tr, m), c)
    sv.build_instance(cost, sv.UniformFrequencies(E), c)
    se.improve_placement(tr, pls[0], cost, iters=2, batch=64)
    with tempfile.TemporaryDirectory() as dd:
        f = os.path.join(dd, "t.txt")
        mt.write_trace(tr.view(2, 9), f, engine="cuda")
        mt.parse_trace(f)
torch.cuda.synchronize()
print("sanitize_all done")
