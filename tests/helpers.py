"""Shared test helpers: seeded inputs, and oracle-side restatements of the product's inputs."""
import numpy as np

import moeplace.model_trace as mt
import moeplace.placement as mpl
import moeplace.topology as topo
from oracle import evaluate as oe
from oracle import topology as ot

R1 = (58, 256, 8)
B16 = (27, 64, 6)


def random_assign(rng, L, E, S, c_layer=None):
    """Feasible-ish random placement: each layer spreads its experts over devices."""
    reps = max(1, -(-E // S))
    out = np.empty((L, E), dtype=np.int32)
    for l in range(L):
        pool = np.repeat(np.arange(S), reps)
        out[l] = rng.permutation(pool)[:E]
    return out


def oracle_cost(g: "topo.ClusterGraph", attn: "mt.AttentionPlacement"):
    dsrv = ot.server_hops(g.n_nodes, g.links.tolist(), g.n_servers)
    return dsrv, ot.cost_matrix(dsrv, g.device_server, attn.dispatch, attn.collect)


def setup_topology(kind, leaves, spl, gps, model, extra=None):
    spec = topo.TopologySpec(kind, leaves, spl, gps, dict(extra or {}))
    g = topo.build_topology(spec)
    dist = topo.all_pairs_hops(g)
    order = topo.locality_order(g, dist)
    attn = mt.default_attention_placement(model, order)
    cost = mpl.cost_matrix(dist, attn)
    return g, dist, order, attn, cost


def oracle_sums(sel, p, assign, bounds, t0=0):
    return oe.chunk_sums(sel, oe.pe_table(p, assign), bounds, t0)
