"""Property tests of the device path (SPEC.md invariants) over random shapes with
hypothesis: every property is checked on the GPU engine's integers/floats."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import moeplace.eval as ev
import moeplace.model_trace as mt
import moeplace.placement as mpl

from helpers import random_assign

pytestmark = pytest.mark.gpu

SETTINGS = dict(max_examples=12, deadline=None, suppress_health_check=[HealthCheck.too_slow])


@st.composite
def case(draw):
    L = draw(st.integers(1, 6))
    E = draw(st.sampled_from([2, 5, 16, 64, 256]))
    K = draw(st.integers(1, min(E, 9)))
    N = draw(st.integers(1, 700))
    C = draw(st.integers(1, 12))
    seed = draw(st.integers(0, 2 ** 31))
    s = draw(st.sampled_from([0.0, 1.2, 2.0]))
    return L, E, K, N, C, seed, s


def _cost(rng, L, S, hi=9):
    import torch
    p = rng.integers(0, hi + 1, (L, S)).astype(np.uint8)
    return mpl.CostMatrix(torch.as_tensor(p, device="cuda")), p


@settings(**SETTINGS)
@given(case())
def test_permutation_within_chunks_and_duplication(c):
    """SPEC.md:382 (permutation within chunks) and SPEC.md:352 (duplicating every token)."""
    L, E, K, N, C, seed, s = c
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, s, N, C, seed)
    sel = tr.tokens()
    lab = tr.token_chunk_ids()
    rng = np.random.default_rng(seed % 1000)
    cost, p = _cost(rng, L, 8)
    pl = mpl.Placement(random_assign(rng, L, E, 8))
    base = ev.evaluate(tr, pl, cost)
    perm = rng.permutation(N)  # from_tokens regroups stably by chunk: a within-chunk shuffle
    shuffled = mt.ActivationTrace.from_tokens(m, sel[perm], lab[perm])
    r2 = ev.evaluate(shuffled, pl, cost)
    nonempty = [x for x, n in zip(base.chunk_hop_sums, tr.chunk_token_counts()) if n > 0]
    assert r2.chunk_hop_sums == nonempty
    assert r2.mean_hops_per_token == base.mean_hops_per_token
    dup = mt.ActivationTrace.from_tokens(m, np.concatenate([sel, sel]), np.concatenate([lab, lab]))
    r3 = ev.evaluate(dup, pl, cost)
    assert r3.mean_hops_per_token == base.mean_hops_per_token
    assert r3.chunk_hop_sums == [2 * x for x in nonempty]


@settings(**SETTINGS)
@given(case())
def test_frequency_invariants(c):
    """rows sum to 1; estimate of a concatenation = count-weighted average."""
    L, E, K, N, C, seed, s = c
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, s, N, C, seed)
    f = mt.estimate_frequencies(tr, m)
    assert np.allclose(f.f.sum(axis=1), 1.0, atol=1e-9)
    if C >= 2 and tr.chunk_bounds[1] > 0 and tr.chunk_bounds[1] < N:
        a, b = tr.view(0, 1), tr.view(1, C)
        fa, fb = mt.estimate_frequencies(a, m), mt.estimate_frequencies(b, m)
        w = (fa.f * a.n_tokens + fb.f * b.n_tokens) / N
        assert np.allclose(w, f.f, rtol=0, atol=1e-12)
        assert np.array_equal(fa.counts + fb.counts, f.counts)


@settings(**SETTINGS)
@given(case())
def test_metric_objective_identity(c):
    """SPEC.md:383 / acceptance #2: evaluate(train).mean == K * objective_value(f_train) (1e-6),
    and the integer form sum(counts * pe) == hop_sum exactly."""
    L, E, K, N, C, seed, s = c
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, s, N, C, seed)
    rng = np.random.default_rng(seed % 977)
    cost, p = _cost(rng, L, 16, hi=30)
    pl = mpl.Placement(random_assign(rng, L, E, 16))
    rep = ev.evaluate(tr, pl, cost)
    f = mt.estimate_frequencies(tr, m)
    obj = ev.objective_value(pl, f, cost)
    assert abs(rep.mean_hops_per_token - K * obj) <= 1e-6 * max(1.0, rep.mean_hops_per_token)
    pe = p.astype(np.int64)[np.arange(L)[:, None], pl.assign]
    assert int((f.counts * pe).sum()) == rep.hop_sum
    assert np.array_equal(ev.token_hops_all(tr, [pl], cost)[0].sum(), rep.hop_sum)


@settings(max_examples=6, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(0, 2 ** 31), st.sampled_from(["FatTree", "FatTreeHier", "Dragonfly", "DragonflySparse"]))
def test_commmap_mass_equals_mean(seed, kind):
    """CommMap total mass == evaluate mean; symmetric, zero diagonal."""
    from helpers import setup_topology
    m = mt.ModelSpec(5, 32, 3)
    g, dist, order, attn, cost = setup_topology(kind, 4, 2, 2, m)
    tr = mt.generate_trace(m, 1.2, 900, 6, seed)
    pl = mpl.Placement(random_assign(np.random.default_rng(seed % 101), 5, 32, g.n_devices))
    cm = ev.communication_map(tr, pl, cost)
    rep = ev.evaluate(tr, pl, cost)
    assert abs(cm.traffic.sum() - rep.mean_hops_per_token) <= 1e-9 * max(1.0, rep.mean_hops_per_token)
    assert np.allclose(cm.traffic, cm.traffic.T) and (np.diag(cm.traffic) == 0).all()


@settings(**SETTINGS)
@given(case(), st.sampled_from([1, 2, 4]), st.sampled_from([9, 31, 63, 255]), st.integers(1, 40))
def test_gather_and_count_contract_agree(c, W, hi, S):
    """The three exact hop-sum algorithms (per-byte gather, count-contract, token-tiled) and the
    oracle agree on random shapes, table widths and cost ranges, with and without the histogram."""
    from oracle import evaluate as oe
    from oracle import stats as ost
    L, E, K, N, C, seed, s = c
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, s, N, C, seed)
    sel = tr.tokens()
    rng = np.random.default_rng(seed % 997)
    cost, p = _cost(rng, L, S, hi)
    pls = [mpl.Placement(rng.integers(0, S, (L, E)).astype(np.int32)) for _ in range(4 * W)]
    want = np.stack([oe.chunk_sums(sel, oe.pe_table(p, pl.assign), tr.chunk_bounds) for pl in pls])
    seg = ("seg",) if K == 8 and hi <= 31 else ()
    for algo in ("gather", "count", "token") + seg:
        assert np.array_equal(ev.score_sums(tr, pls, cost, algo=algo), want), algo
    n = 4 if W == 1 else 4 * W
    for algo in ("count", "token") + seg:
        f, reps = ev.evaluate_with_stats(tr, pls[:n], cost, algo=algo)
        assert np.array_equal(f.counts, ost.counts(sel, E))
        assert [r.chunk_hop_sums for r in reps] == want[:n].tolist()


@st.composite
def big_case(draw):
    L = draw(st.integers(1, 8))
    E = draw(st.sampled_from([16, 64, 256]))
    K = draw(st.sampled_from([1, 2, 3, 5, 6, 7, 8, 8, 8]))
    N = draw(st.integers(5_000, 300_000))
    C = draw(st.integers(1, 5_000))
    return L, E, K, N, C, draw(st.integers(0, 2 ** 31)), draw(st.sampled_from([0.0, 1.2, 2.0]))


@settings(max_examples=int(__import__("os").environ.get("MP_STRESS_EXAMPLES", "8")), deadline=None,
          suppress_health_check=[HealthCheck.too_slow])
@given(big_case(), st.sampled_from([1, 2, 4]))
def test_pipelined_flush_multi_cta_stress(c, W):
    """Many CTAs, pieces cut by chunk and CTA boundaries, 1-5000 chunks: the pipelined-flush
    count-contract (three rotating replica sets, per-set mbarriers) and per-chunk histogram equal
    the per-byte gather and numpy on the same trace."""
    L, E, K, N, C, seed, s = c
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, s, N, C, seed)
    rng = np.random.default_rng(seed % 991)
    cost, p = _cost(rng, L, 23, 31)
    pls = [mpl.Placement(rng.integers(0, 23, (L, E)).astype(np.int32)) for _ in range(4 * W)]
    want = ev.score_sums(tr, pls, cost, algo="gather")
    assert np.array_equal(ev.score_sums(tr, pls, cost, algo="count"), want)
    if K == 8:  # segmented gather: warp ranges and chunk boundaries at every position
        assert np.array_equal(ev.score_sums(tr, pls, cost, algo="seg"), want)
        if W == 1:
            f2, r2 = ev.evaluate_with_stats(tr, pls, cost, algo="seg")
            assert [r.chunk_hop_sums for r in r2] == want.tolist()
    f, reps = ev.evaluate_with_stats(tr, pls[:4 * W], cost, algo="count")
    sel = tr.tokens()
    hist = np.stack([np.bincount(sel[:, l, :].ravel(), minlength=E) for l in range(L)])
    assert np.array_equal(f.counts, hist)
    assert [r.chunk_hop_sums for r in reps] == want.tolist()
    cc = mt.chunk_counts(tr).cpu().numpy()  # per-chunk histogram (pipelined flush, WC = 0)
    assert np.array_equal(cc.sum(axis=0), hist)
    b = tr.chunk_bounds
    for c_ in sorted({0, tr.n_chunks // 2, tr.n_chunks - 1}):
        part = sel[b[c_]:b[c_ + 1]]
        assert np.array_equal(cc[c_], np.stack([np.bincount(part[:, l, :].ravel(), minlength=E) for l in range(L)]))


@settings(max_examples=int(__import__("os").environ.get("MP_STRESS_EXAMPLES", "6")), deadline=None,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(1, 6), st.sampled_from([16, 64, 256]), st.integers(2_000, 60_000), st.integers(1, 3_000),
       st.integers(0, 2 ** 31), st.sampled_from([("FatTree", (4, 2, 4)), ("Dragonfly", (4, 2, 4)),
                                                 ("DragonflySparse", (64, 1, 1))]))
def test_dedup_warp_ranges_stress(L, E, N, C, seed, topo_case):
    """Unique-destination scoring (K = 8 warp-range path) over many CTAs, warp ranges and chunk
    boundaries at every position, fast (pe <= 31, ids < 128) and general layers: bit-exact vs the
    oracle."""
    from helpers import oracle_cost, setup_topology
    from oracle import evaluate as oe
    from oracle import gen as og
    kind, size = topo_case
    m = mt.ModelSpec(L, E, 8)
    g, dist, order, attn, cost = setup_topology(kind, *size, m)
    _, p = oracle_cost(g, attn)
    tr = mt.generate_trace(m, 1.2, N, C, seed)
    sel, bounds = og.generate(L, E, 8, 1.2, N, C, seed)
    rng = np.random.default_rng(seed % 977)
    pls = [mpl.Placement(random_assign(rng, L, E, g.n_devices)) for _ in range(4)]
    reps = ev.evaluate_dedup(tr, pls, cost)
    src = g.device_server[attn.dispatch]
    for pl, rep in zip(pls, reps):
        h, u, d = oe.dedup_sums(sel, oe.pe_table(p, pl.assign), g.device_server[pl.assign], src, bounds)
        assert rep.spec.chunk_hop_sums == h.tolist()
        assert rep.chunk_uniq_sums == u.tolist()
        assert rep.chunk_dedup_sums == d.tolist()


@settings(max_examples=int(__import__("os").environ.get("MP_STRESS_EXAMPLES", "8")), deadline=None,
          suppress_health_check=[HealthCheck.too_slow])
@given(st.integers(1, 6), st.sampled_from([16, 256]), st.integers(20_000, 200_000), st.integers(2, 4_000),
       st.integers(0, 2 ** 31), st.sampled_from([1, 2, 4]), st.floats(0.0, 0.45), st.floats(0.55, 1.0))
def test_segmented_gather_views_stress(L, E, N, C, seed, W, lo, hi):
    """The segmented gather (round-2 kernel: compile-time interior windows, edge windows only at a
    warp range's odd first token and its end) and the unique-destination kernel on chunk-range VIEWS
    starting and ending at arbitrary (often odd) tokens, over many CTAs: bit-exact against the
    per-byte gather, the oracle histogram and the dedup oracle."""
    from helpers import oracle_cost, setup_topology
    from oracle import evaluate as oe
    m = mt.ModelSpec(L, E, 8)
    tr = mt.generate_trace(m, 1.2, N, C, seed)
    c0, c1 = int(lo * C), max(int(lo * C) + 1, int(hi * C))
    sub = tr.view(c0, c1)
    rng = np.random.default_rng(seed % 983)
    cost, p = _cost(rng, L, 19, 31)
    pls = [mpl.Placement(rng.integers(0, 19, (L, E)).astype(np.int32)) for _ in range(4 * W)]
    want = ev.score_sums(sub, pls, cost, algo="gather")
    assert np.array_equal(ev.score_sums(sub, pls, cost, algo="seg"), want)
    f, reps = ev.evaluate_with_stats(sub, pls, cost, algo="seg")
    sel = sub.tokens()
    assert np.array_equal(f.counts, np.stack([np.bincount(sel[:, l, :].ravel(), minlength=E) for l in range(L)]))
    assert [r.chunk_hop_sums for r in reps] == want.tolist()
    # unique destinations on the same view (FatTree: fast layers)
    g, dist, order, attn, cst = setup_topology("FatTree", 4, 2, 4, m)
    _, pc = oracle_cost(g, attn)
    dp = [mpl.Placement(rng.integers(0, g.n_devices, (L, E)).astype(np.int32)) for _ in range(4)]
    dreps = ev.evaluate_dedup(sub, dp, cst)
    b = sub.chunk_bounds - sub.chunk_bounds[0]
    for pl, rep in zip(dp, dreps):
        h, u, d = oe.dedup_sums(sel, oe.pe_table(pc, pl.assign), g.device_server[pl.assign],
                                g.device_server[attn.dispatch], b)
        assert rep.spec.chunk_hop_sums == h.tolist()
        assert rep.chunk_uniq_sums == u.tolist() and rep.chunk_dedup_sums == d.tolist()
