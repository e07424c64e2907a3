"""Probe (not product code): host-side cost of evaluate_many(method="auto") for 4096 candidate
placements on a 1M-token host trace (config 4 shape): placement tables, the streamed per-chunk
histogram, the contraction and the report construction, each timed alone."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import moeplace.eval as ev  # noqa: E402
import moeplace.model_trace as mt  # noqa: E402
import moeplace.placement as mpl  # noqa: E402
import moeplace.topology as topo  # noqa: E402

m = mt.ModelSpec(58, 256, 8)
g = topo.build_topology(topo.TopologySpec("Dragonfly", 16, 4, 4))
d = topo.all_pairs_hops(g)
order = topo.locality_order(g, d)
attn = mt.default_attention_placement(m, order)
cost = mpl.cost_matrix(d, attn)
c = mpl.Constraints(64, 1)
base = mpl.place_round_robin(m, attn, order, c)
cand = mpl.perturb_swaps(base, 4096, 64, 1000)
pls = [mpl.Placement(cand[i], c, f"cand{i}") for i in range(cand.shape[0])]
tr = mt.generate_trace(m, 1.2, 1_000_000, 150, 0)
host = tr.to_host(pin=True)


def t(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    print(f"{name:40s} {(time.perf_counter() - a) / reps * 1e3:9.2f} ms")
    return r


t("evaluate_many(host, auto)", lambda: ev.evaluate_many(host, pls, cost))
t("evaluate_many(device, auto)", lambda: ev.evaluate_many(tr, pls, cost))
t("  _stack_assign", lambda: ev._stack_assign(pls, [cost] * len(pls), m))
t("  pe_matrix", lambda: ev.pe_matrix(pls, cost, m))
t("  chunk_counts(host)", lambda: mt.chunk_counts(host))
t("  chunk_counts(device)", lambda: mt.chunk_counts(tr))
cnt = mt.chunk_counts(tr)
pe = ev.pe_matrix(pls, cost, m)
t("  contract_tc", lambda: ev.contract_tc(cnt.view(150, -1), pe))
sums = ev.contract_tc(cnt.view(150, -1), pe).cpu().numpy()
tok = tr.chunk_token_counts()
t("  reports", lambda: [ev.report_from_sums(sums[i], tok, pls[i].label) for i in range(len(pls))])
t("  Placement construction x4096", lambda: [mpl.Placement(cand[i], c, f"cand{i}") for i in range(cand.shape[0])], reps=1)
