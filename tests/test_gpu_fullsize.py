"""BASELINE configs at their stated sizes, bit-exact against the CPU oracle (SPEC.md:140-148,
345-353, 383, 446).

The oracle regenerates every token on the CPU with its own sampler restatement (oracle/gen.py),
so each test checks the device generator, the statistics and the scorer at full size, on the
real pipeline placements (RR, Greedy, ILP, ILPLoad from the host placers and the exact solver).
Per-chunk sums are additive over token ranges, so the oracle evaluates large ranges as a few
sub-ranges (``t0``) instead of materialising one copy.
"""
import numpy as np
import pytest

import moeplace.cli as cli
import moeplace.eval as ev
import moeplace.model_trace as mt
import moeplace.placement as mpl
import moeplace.solver as sv
from oracle import evaluate as oe
from oracle import gen as og
from oracle import stats as ost

from helpers import oracle_cost, setup_topology

pytestmark = pytest.mark.gpu

L, E, K = 58, 256, 8
N2, C2 = 10_000_000, 150          # config 2 / 3: R1, 10M tokens, 150 chunks, Zipf 1.2, seed 0
N5, C5 = 100_000_000, 1500        # config 5: 100M tokens, 1500 chunks
SUB5 = (5_000_000, 15_000_000)    # config 5 oracle sub-range (crosses the 8-shard boundary at 12.5M)
MODEL = mt.ModelSpec(L, E, K)
CONS = mpl.Constraints(64, 1)


def _methods(freq, topo_tuple, label):
    g, dist, order, attn, cost = topo_tuple
    out = [mpl.place_round_robin(MODEL, attn, order, CONS), mpl.place_greedy(MODEL, attn, cost, CONS),
           sv.solve_exact(sv.build_instance(cost, sv.UniformFrequencies(E), CONS))[0],
           sv.solve_exact(sv.build_instance(cost, freq, CONS))[0]]
    for pl, m in zip(out, ("rr", "greedy", "ilp", "ilpload")):
        pl.label = f"{label}/{m}"
    return out


@pytest.fixture(scope="module")
def oracle_r1():
    """Oracle tokens [0, 10M) of the seed-0 R1 trace (shared by configs 2, 3 and 5: the sampler
    depends on (seed, token, layer) only, not on N or C)."""
    sel, _ = og.generate(L, E, K, 1.2, N2, C2, 0)
    return sel


@pytest.fixture(scope="module")
def config2(oracle_r1):
    tr = mt.generate_trace(MODEL, 1.2, N2, C2, 0)
    freq = mt.estimate_frequencies(tr, MODEL)
    ft = setup_topology("FatTree", 8, 4, 8, MODEL, {"spines": 4})
    pls = _methods(freq, ft, "FatTree")
    return tr, freq, ft, pls


def test_config2_generator_full_size(config2, oracle_r1):
    """Every byte of the 10M-token device trace equals the oracle's (compared on the device)."""
    import torch
    tr = config2[0]
    want = torch.from_numpy(oracle_r1).to(tr.planes.device)       # token-major [N, L, K]
    got = tr.planes[:, :N2 * K].view(L, N2, K).permute(1, 0, 2)
    assert torch.equal(got, want)
    assert np.array_equal(tr.chunk_bounds, mt.chunk_bounds_even(N2, C2))


def test_config2_full_size_counts_and_hop_sums(config2, oracle_r1):
    """BASELINE config 2 (the benched step): load counts [58 x 256] and the per-chunk hop sums
    [4 x 150] of the real RR / Greedy / ILP / ILPLoad placements over all 10M tokens, through the
    fused pass (AUTO = count-contract, pipelined flush) and every explicit algorithm."""
    tr, freq, ft, pls = config2
    g, dist, order, attn, cost = ft
    dsrv, p = oracle_cost(g, attn)
    assert np.array_equal(cost.numpy(), p)
    bounds = mt.chunk_bounds_even(N2, C2)
    want_cnt = ost.counts(oracle_r1, E)
    assert np.array_equal(freq.counts, want_cnt)
    pes = [oe.pe_table(p, pl.assign) for pl in pls]
    want = np.stack([oe.chunk_sums(oracle_r1, pe, bounds) for pe in pes])
    # the oracle's one-pass form (the CPU baseline) agrees with its per-chunk loops at full size
    f_cnt, f_sums = oe.fused_pass(oracle_r1, pes, bounds, E)
    assert np.array_equal(f_cnt, want_cnt) and np.array_equal(f_sums, want)
    f, reps = ev.evaluate_with_stats(tr, pls, cost)               # AUTO: count-contract (bench step)
    assert np.array_equal(f.counts, want_cnt)
    assert np.array_equal(np.array([r.chunk_hop_sums for r in reps]), want)
    tok = np.diff(bounds)
    for i, r in enumerate(reps):
        o = oe.report(want[i], tok)
        assert (r.mean_hops_per_token, r.std_hops, r.hop_sum) == (o["mean"], o["std"], o["hop_sum"])
    for algo in ("gather", "count", "token", "seg"):
        assert np.array_equal(ev.score_sums(tr, pls, cost, algo=algo), want), algo
        f, reps = ev.evaluate_with_stats(tr, pls, cost, algo=algo)
        assert np.array_equal(f.counts, want_cnt), algo
        assert np.array_equal(np.array([r.chunk_hop_sums for r in reps]), want), algo
    assert np.array_equal(ev.score_sums_factorized(tr, pls, cost), want)
    # acceptance #2 on the full trace: mean == K * objective
    fr = mt.frequencies_from_counts(want_cnt, N2, K)
    for pl, r in zip(pls, ev.evaluate_many(tr, pls, cost)):
        obj = ev.objective_value(pl, fr, cost)
        assert abs(r.mean_hops_per_token - K * obj) <= 1e-9 * r.mean_hops_per_token


def test_config3_six_topologies_full_size(config2, oracle_r1):
    """BASELINE config 3: R1 at 10M tokens on FatTree, FatTreeHier, Dragonfly, DragonflySparse,
    DragonflyPlus (16 x 4 x 4) and SlimFly (18 leaves x 4 x 4) -- 24 placements (4 methods each)
    scored as one 32-lane count-contract pass (what AUTO runs) and factorized, against the oracle."""
    tr, freq = config2[0], config2[1]
    bounds = mt.chunk_bounds_even(N2, C2)
    pls, costs, pes = [], [], []
    for kind, leaves in (("FatTree", 16), ("FatTreeHier", 16), ("Dragonfly", 16), ("DragonflySparse", 16),
                         ("DragonflyPlus", 16), ("SlimFly", 18)):
        tt = setup_topology(kind, leaves, 4, 4, MODEL)
        g, attn, cost = tt[0], tt[3], tt[4]
        _, p = oracle_cost(g, attn)
        assert np.array_equal(cost.numpy(), p), kind
        for pl in _methods(freq, tt, kind):
            assert mpl.validate(pl, CONS, MODEL, g.n_devices) == [], pl.label
            pls.append(pl)
            costs.append(cost)
            pes.append(oe.pe_table(p, pl.assign))
    _, want = oe.fused_pass(oracle_r1, pes, bounds, E)
    assert ev.pass_lanes(tr, costs) == 32
    for method in ("factorized", "auto"):
        reps = ev.evaluate_many(tr, pls, costs, method=method)
        assert np.array_equal(np.array([r.chunk_hop_sums for r in reps]), want), method
    # ILPLoad is the best of the four methods on every topology (train == test == full trace here)
    means = np.array([r.mean_hops_per_token for r in reps]).reshape(6, 4)
    assert (means[:, 3] <= means.min(axis=1) + 1e-12).all()


def test_config5_sharded_100m_against_oracle_subrange(config2, oracle_r1):
    """BASELINE config 5: the 100M-token trace (1500 chunks) sharded over G = 1, 2, 4, 8 (emulated
    on one GPU: each rank's shard generated, evaluated and its packed partials summed, which is
    what the NCCL all_reduce does).  The integers are identical for every G, and a 10M-token
    sub-range crossing a shard boundary is bit-exact against the oracle."""
    import torch
    from paper_2508_09229_b200.shard import shard_range, sharded_evaluate
    pls, ft = config2[3], config2[2]
    cost = ft[4]
    res = {}
    for G in (1, 2, 4, 8):
        cnt = np.zeros((L, E), np.int64)
        sums = np.zeros((len(pls), C5), np.int64)
        for r in range(G):
            f, reps = sharded_evaluate(MODEL, 1.2, N5, C5, 0, pls, cost, rank=r, world=G)
            cnt += f.counts
            sums += np.array([x.chunk_hop_sums for x in reps])
            torch.cuda.empty_cache()
        res[G] = (cnt, sums)
    for G in (2, 4, 8):
        assert np.array_equal(res[G][0], res[1][0]) and np.array_equal(res[G][1], res[1][1]), G
    assert (res[1][0].sum(axis=1) == N5 * K).all()
    # oracle on [5M, 15M): tokens [5M, 10M) from the shared fixture, [10M, 15M) regenerated
    a, b = SUB5
    sel_b, bounds = og.generate(L, E, K, 1.2, N5, C5, 0, tok_range=(N2, b))
    _, p = oracle_cost(ft[0], ft[3])
    want = np.zeros((len(pls), C5), np.int64)
    want_cnt = ost.counts(oracle_r1[a:], E) + ost.counts(sel_b, E)
    for i, pl in enumerate(pls):
        pe = oe.pe_table(p, pl.assign)
        want[i] = oe.chunk_sums(oracle_r1[a:], pe, bounds, a) + oe.chunk_sums(sel_b, pe, bounds, N2)
    sub = mt.generate_trace(MODEL, 1.2, N5, C5, 0, tok_range=SUB5)
    f, reps = ev.evaluate_with_stats(sub, pls, cost)
    assert np.array_equal(f.counts, want_cnt)
    assert np.array_equal(np.array([r.chunk_hop_sums for r in reps]), want)
    # the sub-range is exactly the sum of the 8-shard partials restricted to it
    parts = np.zeros_like(want)
    for r in range(8):
        s0, s1 = shard_range(N5, r, 8)
        lo, hi = max(s0, a), min(s1, b)
        if lo < hi:
            v = mt.generate_trace(MODEL, 1.2, N5, C5, 0, tok_range=(lo, hi))
            parts += ev.score_sums(v, pls, cost)
    assert np.array_equal(parts, want)


def test_sharded_evaluate_every_rank_short_chunks():
    """sharded_evaluate for every rank of an 8-way split where shards start mid-chunk,
    leading chunks are empty for a shard, and AUTO sees shard-sized inputs against the global C
    (picking SEG / TOKEN): the rank partials sum to the one-GPU pass and to the oracle."""
    from paper_2508_09229_b200.shard import sharded_evaluate
    N, C = 200_003, 3001                      # ~67 tokens per chunk: TOKEN / SEG territory
    ft = setup_topology("FatTree", 8, 4, 8, MODEL, {"spines": 4})
    g, dist, order, attn, cost = ft
    pls = [mpl.place_round_robin(MODEL, attn, order, CONS), mpl.place_greedy(MODEL, attn, cost, CONS)]
    cnt = np.zeros((L, E), np.int64)
    sums = np.zeros((2, C), np.int64)
    for r in range(8):
        f, reps = sharded_evaluate(MODEL, 1.2, N, C, 3, pls, cost, rank=r, world=8)
        cnt += f.counts
        sums += np.array([x.chunk_hop_sums for x in reps])
    tr = mt.generate_trace(MODEL, 1.2, N, C, 3)
    f1, r1 = ev.evaluate_with_stats(tr, pls, cost)
    assert np.array_equal(cnt, f1.counts)
    assert np.array_equal(sums, np.array([x.chunk_hop_sums for x in r1]))
    sel, bounds = og.generate(L, E, K, 1.2, N, C, 3)
    _, p = oracle_cost(g, attn)
    assert np.array_equal(cnt, ost.counts(sel, E))
    for i, pl in enumerate(pls):
        assert np.array_equal(sums[i], oe.chunk_sums(sel, oe.pe_table(p, pl.assign), bounds))
    # the floats of the combined partials are the one-GPU report floats
    rep = ev.reports_from_sums(sums, np.diff(bounds), ["rr", "greedy"])
    assert [(x.mean_hops_per_token, x.std_hops) for x in rep] == [(x.mean_hops_per_token, x.std_hops) for x in r1]


def test_config1_run_experiment_1m_equals_oracle(tmp_path):
    """BASELINE config 1 at its stated 1M tokens (16B shape, FatTree 2 leaves x 2 servers x 8 GPUs,
    c_layer 2, c_exp 54, 150 chunks, 100/50 split) through run_experiment: the comparison CSV is
    byte-identical to the one rebuilt from the CPU oracle, and the ILPLoad frequencies are the
    oracle's train-split counts."""
    cfg = {"model": "16b", "L": 27, "E": 64, "K": 6, "c_exp": 54, "c_layer": 2, "topology": "FatTree",
           "num_leaf_switches": 2, "num_nodes_per_leaf": 2, "num_gpus_per_server": 8, "spines": 4,
           "zipf_s": 1.2, "n_tokens": 1_000_000, "n_chunks": 150, "seed": 0, "train_chunks": 100,
           "test_chunks": 50, "output_dir": str(tmp_path / "c1")}
    cli.run_experiment(cfg)
    out = tmp_path / "c1"
    model = mt.ModelSpec(27, 64, 6)
    sel, bounds = og.generate(27, 64, 6, 1.2, 1_000_000, 150, 0)
    g, dist, order, attn, cost = setup_topology("FatTree", 2, 2, 8, model, {"spines": 4})
    _, p = oracle_cost(g, attn)
    tok = np.diff(bounds)
    rows, base = [], None
    for m in ("rr", "greedy", "ilp", "ilpload"):
        asg = mpl.read_placement(out / f"placement_{m}.csv", model).assign
        sums = oe.chunk_sums(sel, oe.pe_table(p, asg), bounds)
        r = oe.report(sums[100:150], tok[100:150])
        if m == "rr":
            base = r["mean"]
        rows.append(f"FatTree,{m},{r['mean']!r},{r['std']!r},{oe.gain(base, r['mean'])!r}\n")
    want = "network,placement,hops_mean,hops_std,gain_pct\n" + "".join(rows)
    assert (out / "comparison.csv").read_text() == want
    # the ILPLoad instance is built from the train split's counts: re-solve from the oracle's counts
    train_cnt = ost.counts(sel[:bounds[100]], 64)
    fr = mt.frequencies_from_counts(train_cnt, int(bounds[100]), 6)
    ilpload = sv.solve_exact(sv.build_instance(cost, fr, mpl.Constraints(54, 2)))[0]
    assert np.array_equal(ilpload.assign, mpl.read_placement(out / "placement_ilpload.csv", model).assign)
