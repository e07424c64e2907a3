"""The two exact hop-sum algorithms behind mp_score_u8 / mp_hist_score_u8 (per-byte GATHER and
COUNT-contract, include/moeplace_cuda.h) are bit-identical to each other and to the oracle
(oracle/evaluate.py chunk_sums, oracle/stats.py counts) for every table width, on sub-ranges,
empty chunks, pieces above the 16 MB contract cap, large costs and out-of-range ids."""
import numpy as np
import pytest

import moeplace.eval as ev
import moeplace.model_trace as mt
import moeplace.placement as mpl
from oracle import gen as og
from oracle import stats as ost

from helpers import B16, R1, oracle_sums, random_assign

pytestmark = pytest.mark.gpu

AUTO, GATHER, COUNT, TOKEN, SEG = 0, 1, 2, 3, 4


def _tables(pls, p, m, W):
    import torch
    cost = mpl.CostMatrix(torch.as_tensor(p, device="cuda"))
    return ev._group_tables(pls, [cost] * len(pls), m, W)


def _run(tr, tables, W, max_p, algo, hist):
    import torch
    from paper_2508_09229_b200 import _lib
    m = tr.model
    C = len(tr.chunk_bounds) - 1
    bounds = _lib.to_dev(tr.chunk_bounds, torch.int64)
    sums = torch.zeros((4 * W, C), dtype=torch.int64, device="cuda")
    counts = torch.zeros((m.L, m.E), dtype=torch.int64, device="cuda")
    err = _lib.new_err()
    stride = tr.planes.shape[1]
    if hist:
        _lib.call("mp_hist_score_ex_u8", _lib.ptr(tr.planes), stride, tr.tok_begin, tr.tok_end, m.L, m.K, m.E,
                  _lib.ptr(bounds), C, _lib.ptr(tables), W, max_p, _lib.ptr(counts), _lib.ptr(sums), _lib.ptr(err),
                  algo, _lib.stream_handle())
    else:
        _lib.call("mp_score_ex_u8", _lib.ptr(tr.planes), stride, tr.tok_begin, tr.tok_end, m.L, m.K,
                  _lib.ptr(bounds), C, _lib.ptr(tables), W, max_p, _lib.ptr(sums), algo, _lib.stream_handle())
    torch.cuda.synchronize()
    return sums.cpu().numpy(), counts.cpu().numpy(), _lib.read_err(err)


def _check(tr, sel, bounds, t0, pls, p, W, hist_ws=(1,)):
    m = tr.model
    tables, max_p = _tables(pls, p, m, W)
    want = np.zeros((4 * W, len(bounds) - 1), np.int64)
    for i, pl in enumerate(pls):
        want[i] = oracle_sums(sel, p, pl.assign, bounds, t0)
    algos = (AUTO, GATHER, COUNT) + ((TOKEN,) if m.L * m.K * max_p <= 65535 else ()) + \
        ((SEG,) if m.K == 8 and max_p <= 31 else ())
    for algo in algos:
        s, _, _ = _run(tr, tables, W, max_p, algo, hist=False)
        assert np.array_equal(s, want), ("score", W, algo)
        if W in hist_ws or algo != GATHER:
            s, c, e = _run(tr, tables, W, max_p, algo, hist=True)
            assert np.array_equal(s, want), ("hist_score", W, algo)
            assert np.array_equal(c, ost.counts(sel, m.E)), ("counts", W, algo)
            assert e[0] == 0


@pytest.mark.parametrize("W", [1, 2, 4])
@pytest.mark.parametrize("shape", [R1, B16, (3, 5, 2), (5, 200, 7)])
@pytest.mark.parametrize("cmax", [13, 32])
def test_algorithms_agree_with_oracle(shape, W, cmax):
    """Costs < 13 take the segmented gather's nibble tables (W = 2 / 4, max_p <= 15); costs up to 31
    its u8 tables."""
    L, E, K = shape
    m = mt.ModelSpec(L, E, K)
    N, C = 5003, 17
    tr = mt.generate_trace(m, 1.2, N, C, 3)
    sel, bounds = og.generate(L, E, K, 1.2, N, C, 3)
    rng = np.random.default_rng(W)
    S = 24
    p = rng.integers(0, cmax, (L, S)).astype(np.uint8)
    pls = [mpl.Placement(random_assign(rng, L, E, S)) for _ in range(4 * W - (1 if W > 1 else 0))]
    _check(tr, sel, bounds, 0, pls, p, W)
    # a chunk sub-range view (token range starts mid-trace; plane byte offsets unaligned)
    sub = tr.view(3, 11)
    a, b = int(bounds[3]), int(bounds[11])
    _check(sub, sel[a:b], bounds[3:12], a, pls, p, W)


@pytest.mark.parametrize("shape", [R1, B16, (5, 200, 7)])
@pytest.mark.parametrize("nplace", [17, 24, 32])
def test_count_contract_32_lanes(shape, nplace):
    """W = 8 (up to 32 placements in one count-contract pass) == the oracle, with and without the
    histogram, on whole traces and on a view; the other algorithms refuse W = 8 explicitly."""
    L, E, K = shape
    m = mt.ModelSpec(L, E, K)
    N, C = 6007, 11
    tr = mt.generate_trace(m, 1.2, N, C, 5)
    sel, bounds = og.generate(L, E, K, 1.2, N, C, 5)
    rng = np.random.default_rng(nplace)
    p = rng.integers(0, 40, (L, 24)).astype(np.uint8)
    pls = [mpl.Placement(random_assign(rng, L, E, 24)) for _ in range(nplace)]
    tables, max_p = _tables(pls, p, m, 8)
    want = np.zeros((32, C), np.int64)
    for i, pl in enumerate(pls):
        want[i] = oracle_sums(sel, p, pl.assign, bounds, 0)
    for algo in (AUTO, COUNT):
        s, _, _ = _run(tr, tables, 8, max_p, algo, hist=False)
        assert np.array_equal(s, want), algo
        s, c, e = _run(tr, tables, 8, max_p, algo, hist=True)
        assert np.array_equal(s, want) and np.array_equal(c, ost.counts(sel, m.E)) and e[0] == 0, algo
    sub = tr.view(2, 9)
    a, b = int(bounds[2]), int(bounds[9])
    s, _, _ = _run(sub, tables, 8, max_p, AUTO, hist=False)
    for i, pl in enumerate(pls):
        assert np.array_equal(s[i], oracle_sums(sel[a:b], p, pl.assign, bounds[2:10], a)), i
    from paper_2508_09229_b200 import _lib
    import torch
    P_ = _lib.ptr(tr.planes)
    for algo in (GATHER, TOKEN, SEG):
        assert _lib.load().mp_score_ex_u8(P_, tr.planes.shape[1], 0, N, L, K, _lib.ptr(_lib.to_dev(tr.chunk_bounds,
                                          torch.int64)), C, _lib.ptr(tables), 8, max_p,
                                          _lib.ptr(torch.zeros((32, C), dtype=torch.int64, device="cuda")), algo,
                                          None) == 3


def test_algorithms_agree_on_empty_chunks_and_large_costs():
    L, E, K = B16
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, 2.0, 90, 150, 1)  # N < C: many empty chunks
    sel, bounds = og.generate(L, E, K, 2.0, 90, 150, 1)
    rng = np.random.default_rng(5)
    p = rng.integers(200, 256, (L, 8)).astype(np.uint8)
    pls = [mpl.Placement(random_assign(rng, L, E, 8)) for _ in range(16)]
    for W in (1, 2, 4):
        _check(tr, sel, bounds, 0, pls[:4 * W], p, W)


def test_count_contract_splits_pieces_above_cap():
    """One layer x one chunk of 24 MB (> the 16 MB contract piece cap), costs up to 255: the
    per-piece u32 partials must not overflow and the split pieces must add up exactly."""
    L, E, K = 1, 256, 8
    m = mt.ModelSpec(L, E, K)
    N = 3_000_001
    tr = mt.generate_trace(m, 0.0, N, 1, 9)
    sel, bounds = og.generate(L, E, K, 0.0, N, 1, 9)
    p = np.full((L, 4), 255, np.uint8)
    p[0, 1] = 254
    rng = np.random.default_rng(0)
    pls = [mpl.Placement(random_assign(rng, L, E, 4)) for _ in range(4)]
    _check(tr, sel, bounds, 0, pls, p, 1)


def test_out_of_range_ids_same_result_both_algorithms():
    """Ids >= E: not counted, reported as MP_DATA_EXPERT_RANGE, and they add 0 hops (table rows
    e >= E are zero) -- identically for both algorithms."""
    import torch
    L, E, K = 4, 40, 4
    m = mt.ModelSpec(L, E, K)
    N, C = 777, 5
    tr = mt.generate_trace(m, 1.2, N, C, 2)
    planes = tr.planes.clone()
    planes[2, 5 * K + 1] = 200  # token 5, layer 2
    planes[0, 700 * K] = 41
    bad = mt.ActivationTrace(m, planes, 0, N, tr.chunk_ids.copy(), tr.chunk_bounds.copy(), _validated=True)
    rng = np.random.default_rng(3)
    p = rng.integers(1, 9, (L, 8)).astype(np.uint8)
    pls = [mpl.Placement(random_assign(rng, L, E, 8)) for _ in range(4)]
    tables, max_p = _tables(pls, p, m, 1)
    res = [_run(bad, tables, 1, max_p, algo, hist=True) for algo in (GATHER, COUNT, TOKEN)]
    for r in res[1:]:
        assert np.array_equal(res[0][0], r[0]) and np.array_equal(res[0][1], r[1])
    for s, c, e in res:
        assert e[0] == 1  # MP_DATA_EXPERT_RANGE
        assert c.sum() == N * L * K - 2
    clean = planes.clone()
    clean[2, 5 * K + 1] = 0
    clean[0, 700 * K] = 0
    sel = clean.cpu().numpy()[:, :N * K].reshape(L, N, K).transpose(1, 0, 2)
    want = np.stack([oracle_sums(sel, p, pl.assign, tr.chunk_bounds) for pl in pls])
    # the oracle sees id 0 where the bad ids were: subtract pe[l][0] for those two picks
    for i, pl in enumerate(pls):
        pe = p[np.arange(L)[:, None], pl.assign]
        want[i, 0] -= pe[2, 0]
        want[i, np.searchsorted(tr.chunk_bounds, 700, side="right") - 1] -= pe[0, 0]
    assert np.array_equal(res[1][0][:4], want)


def test_argument_rules_of_the_explicit_entry_points():
    import torch
    from paper_2508_09229_b200 import _lib
    L = _lib.load()
    x = torch.zeros(64, dtype=torch.uint8, device="cuda")
    P = x.data_ptr()
    assert L.mp_hist_score_ex_u8(P, 64, 0, 8, 1, 8, 256, P, 1, P, 2, 8, P, P, P, GATHER, None) == 3
    assert L.mp_hist_score_ex_u8(P, 64, 0, 8, 1, 8, 256, P, 1, P, 3, 8, P, P, P, COUNT, None) == 1
    assert L.mp_score_ex_u8(P, 64, 0, 8, 1, 8, P, 1, P, 1, 8, P, 7, None) == 1
    # segmented gather: K = 8 and max_p <= 31 only, W = 1 with a histogram
    assert L.mp_score_ex_u8(P, 64, 0, 8, 1, 6, P, 1, P, 1, 8, P, SEG, None) == 3
    assert L.mp_score_ex_u8(P, 64, 0, 8, 1, 8, P, 1, P, 1, 40, P, SEG, None) == 3
    assert L.mp_hist_score_ex_u8(P, 64, 0, 8, 1, 6, 256, P, 1, P, 2, 8, P, P, P, SEG, None) == 3


def test_public_api_algorithms_and_wide_stats_pass():
    """evaluate_many(method=auto|gather|count|factorized) and evaluate_with_stats with up to 16
    placements over mixed topologies: identical integers, equal to the oracle."""
    from moeplace.errors import ConfigError
    from helpers import oracle_cost, setup_topology
    L, E, K = B16
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, 1.2, 3001, 12, 6)
    sel, bounds = og.generate(L, E, K, 1.2, 3001, 12, 6)
    costs, ps, pls = [], [], []
    for i, kind in enumerate(["FatTree", "Dragonfly", "DragonflySparse", "FatTreeHier"]):
        g, dist, order, attn, cost = setup_topology(kind, 4, 2, 4, m)
        _, p = oracle_cost(g, attn)
        for j in range(5):
            pls.append(mpl.Placement(random_assign(np.random.default_rng(10 * i + j), L, E, g.n_devices)))
            costs.append(cost)
            ps.append(p)
    want = np.stack([oracle_sums(sel, p, pl.assign, bounds) for p, pl in zip(ps, pls)])
    for n in (5, 16, 20):
        for method in ("auto", "gather", "count", "factorized"):
            reps = ev.evaluate_many(tr, pls[:n], costs[:n], method=method)
            assert [r.chunk_hop_sums for r in reps] == want[:n].tolist(), (n, method)
    for n in (1, 4, 9, 16):
        for algo in (("auto", "count", "gather") if n <= 4 else ("auto", "count")):
            f, reps = ev.evaluate_with_stats(tr, pls[:n], costs[:n], algo=algo)
            assert np.array_equal(f.counts, ost.counts(sel, E))
            assert [r.chunk_hop_sums for r in reps] == want[:n].tolist(), (n, algo)
    # count-contract passes take 32 placements (W = 8); AUTO on these short chunks takes 16
    f, reps = ev.evaluate_with_stats(tr, pls[:20], costs[:20], algo="count")
    assert np.array_equal(f.counts, ost.counts(sel, E))
    assert [r.chunk_hop_sums for r in reps] == want[:20].tolist()
    assert ev.pass_lanes(tr, costs, "count") == 32 and ev.pass_lanes(tr, costs, "auto") == 16
    with pytest.raises(ConfigError):
        ev.evaluate_with_stats(tr, pls[:5], costs[:5], algo="gather")
    with pytest.raises(ConfigError):
        ev.evaluate_with_stats(tr, pls[:17], costs[:17])
    with pytest.raises(ConfigError):
        ev.evaluate_with_stats(tr, (pls * 2)[:33], (costs * 2)[:33], algo="count")


def test_evaluate_batch_matches_evaluate_many():
    """evaluate_batch (one [P, L, E] array: numpy, torch host/pinned or device) gives the same
    integers and floats as evaluate_many's EvalReports, factorized (P > 16) and per pass, and
    rejects out-of-range devices and bad shapes."""
    import torch
    from moeplace.errors import ConfigError, MoeplaceError
    from helpers import setup_topology
    L, E, K = B16
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, 1.2, 2501, 9, 8)
    g, dist, order, attn, cost = setup_topology("Dragonfly", 4, 2, 4, m)
    base = mpl.place_round_robin(m, attn, order, mpl.Constraints(64, 2))
    cand = mpl.perturb_swaps(base, 21, 5, 300)
    pls = [mpl.Placement(cand[i]) for i in range(cand.shape[0])]
    for n in (21, 6):
        want = ev.evaluate_many(tr, pls[:n], cost)
        for arr in (cand[:n], torch.from_numpy(cand[:n]).pin_memory(), torch.from_numpy(cand[:n]).cuda()):
            for method in ("auto", "factorized", "count"):
                b = ev.evaluate_batch(tr, arr, cost, method=method)
                assert b.chunk_hop_sums.tolist() == [r.chunk_hop_sums for r in want], (n, method)
                assert [b.report(q) for q in range(n)] == [ev.EvalReport(**{**r.__dict__, "label": ""}) for r in want]
    bad = cand[:3].copy()
    bad[1, 2, 3] = g.n_devices
    with pytest.raises(MoeplaceError, match="placement 1"):
        ev.evaluate_batch(tr, bad, cost)
    with pytest.raises(ConfigError):
        ev.evaluate_batch(tr, cand[:, :2], cost)


def test_plane_offsets_beyond_2_pow_31():
    """One plane longer than 2^31 bytes (N*K = 2.4e9): 64-bit byte offsets through every piece
    of both algorithms.  Properties: per-layer counts sum to N*K, constant costs give exactly
    p*N*L*K, gather == count, the histogram.table identity holds, and a CPU-regenerated window
    at the far end of the plane matches the oracle."""
    import torch
    L, E, K = 2, 256, 8
    m = mt.ModelSpec(L, E, K)
    N, C = 300_000_000, 40
    tr = mt.generate_trace(m, 1.2, N, C, 4)
    assert tr.planes.shape[1] >= N * K > 2 ** 31
    rng = np.random.default_rng(2)
    S = 16
    p = rng.integers(0, 40, (L, S)).astype(np.uint8)
    pls = [mpl.Placement(random_assign(rng, L, E, S)) for _ in range(4)]
    tables, max_p = _tables(pls, p, m, 1)
    sg, cg, eg = _run(tr, tables, 1, max_p, GATHER, hist=True)
    sc, cc, ec = _run(tr, tables, 1, max_p, COUNT, hist=True)
    assert eg[0] == 0 and ec[0] == 0
    assert np.array_equal(cg, cc) and (cc.sum(axis=1) == N * K).all()
    assert np.array_equal(sg, sc)
    for i, pl in enumerate(pls):
        pe = p[np.arange(L)[:, None], pl.assign]
        assert int((cc * pe).sum()) == int(sc[i].sum())
    const = np.full((L, S), 7, np.uint8)
    t7, _ = _tables(pls[:1], const, m, 1)
    s7, _, _ = _run(tr, t7, 1, 7, COUNT, hist=False)
    assert int(s7[0].sum()) == 7 * N * L * K
    a, b = N - 20_000, N
    sel, bounds = og.generate(L, E, K, 1.2, N, C, 4, tok_range=(a, b))
    sh = mt.generate_trace(m, 1.2, N, C, 4, tok_range=(a, b))
    assert np.array_equal(sh.tokens(), sel)
    want = oracle_sums(sel, p, pls[0].assign, bounds, a)
    tail = tr.view(C - 1, C)
    tables0, mp0 = _tables(pls[:1], p, m, 1)
    # the last chunk of the big trace, restricted to [a, b): equals the oracle window
    sub = mt.ActivationTrace(m, tail.planes, a, b - a, tail.chunk_ids.copy(),
                             np.array([a, b], dtype=np.int64), _validated=True)
    for algo in (GATHER, COUNT, TOKEN):
        s, _, _ = _run(sub, tables0, 1, mp0, algo, hist=False)
        assert int(s[0].sum()) == int(want.sum()), algo


def test_mixed_topology_sizes_in_one_batch():
    """Cost matrices of different device counts (256 and 64 devices) share one batch: the tables
    are zero-padded to the widest topology and every placement is range-checked against its own."""
    from moeplace.errors import ConfigError, MoeplaceError
    from helpers import oracle_cost, setup_topology
    L, E, K = R1
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, 1.2, 2222, 7, 5)
    sel, bounds = og.generate(L, E, K, 1.2, 2222, 7, 5)
    ga, _, _, attn_a, cost_a = setup_topology("FatTree", 8, 4, 8, m)
    gb, _, _, attn_b, cost_b = setup_topology("Dragonfly", 8, 2, 4, m)
    assert ga.n_devices == 256 and gb.n_devices == 64
    pa, pb = oracle_cost(ga, attn_a)[1], oracle_cost(gb, attn_b)[1]
    rng = np.random.default_rng(4)
    pls, costs, ps, gs = [], [], [], []
    for i in range(6):
        g, c, p = (ga, cost_a, pa) if i % 2 == 0 else (gb, cost_b, pb)
        pls.append(mpl.Placement(random_assign(rng, L, E, g.n_devices)))
        costs.append(c)
        ps.append(p)
        gs.append(g)
    want = np.stack([oracle_sums(sel, p, pl.assign, bounds) for p, pl in zip(ps, pls)])
    for method in ("auto", "gather", "count", "factorized"):
        reps = ev.evaluate_many(tr, pls, costs, method=method)
        assert [r.chunk_hop_sums for r in reps] == want.tolist(), method
    f, reps = ev.evaluate_with_stats(tr, pls, costs)
    assert [r.chunk_hop_sums for r in reps] == want.tolist()
    from oracle import evaluate as oe
    dreps = ev.evaluate_dedup(tr, pls[:4], costs[:4])
    for i in range(4):
        g, c = gs[i], costs[i]
        pe = oe.pe_table(ps[i], pls[i].assign)
        h, u, d = oe.dedup_sums(sel, pe, g.device_server[pls[i].assign], g.device_server[c.attn.dispatch], bounds)
        assert dreps[i].spec.chunk_hop_sums == h.tolist()
        assert dreps[i].chunk_uniq_sums == u.tolist() and dreps[i].chunk_dedup_sums == d.tolist()
    # a device index valid for the 256-device topology but not for the 64-device one
    bad = mpl.Placement(np.full((L, E), 100, np.int32))
    with pytest.raises(MoeplaceError):
        ev.evaluate_many(tr, [pls[0], bad], [cost_a, cost_b])
    with pytest.raises(ConfigError):
        ev.evaluate_many(tr, [mpl.Placement(np.zeros((L, E - 1), np.int32))], cost_a)


@pytest.mark.parametrize("tokens_per_chunk", [1, 3, 31, 33, 700])
@pytest.mark.parametrize("W", [1, 4])
def test_token_algorithm_on_fine_chunks(tokens_per_chunk, W):
    """Chunks of a few tokens: many 32-token warp groups straddle several chunks (segmented scan),
    and AUTO picks the token-tiled algorithm; every algorithm equals the oracle."""
    L, E, K = R1
    m = mt.ModelSpec(L, E, K)
    N = 9001
    C = max(1, N // tokens_per_chunk)
    tr = mt.generate_trace(m, 1.2, N, C, 7)
    sel, bounds = og.generate(L, E, K, 1.2, N, C, 7)
    rng = np.random.default_rng(tokens_per_chunk)
    p = rng.integers(0, 60, (L, 16)).astype(np.uint8)
    pls = [mpl.Placement(random_assign(rng, L, E, 16)) for _ in range(4 * W)]
    _check(tr, sel, bounds, 0, pls, p, W)
    sub = tr.view(C // 3, C - C // 5)
    a = int(bounds[C // 3])
    _check(sub, sel[a:int(bounds[C - C // 5])], bounds[C // 3:C - C // 5 + 1], a, pls, p, W)


def test_token_algorithm_limit():
    """Per-token sums must fit u16 lanes: L*K*max_p > 65535 is refused for TOKEN and avoided by AUTO."""
    import torch
    from paper_2508_09229_b200 import _lib
    L, E, K = R1
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, 1.2, 500, 400, 1)  # fine chunks: AUTO would prefer TOKEN
    sel, bounds = og.generate(L, E, K, 1.2, 500, 400, 1)
    rng = np.random.default_rng(0)
    p = rng.integers(100, 256, (L, 8)).astype(np.uint8)  # 58*8*255 > 65535
    pls = [mpl.Placement(random_assign(rng, L, E, 8)) for _ in range(4)]
    tables, max_p = _tables(pls, p, m, 1)
    with pytest.raises(Exception):
        _run(tr, tables, 1, max_p, TOKEN, hist=False)
    s, _, _ = _run(tr, tables, 1, max_p, AUTO, hist=False)
    want = np.stack([oracle_sums(sel, p, pl.assign, bounds) for pl in pls])
    assert np.array_equal(s, want)


def test_evaluate_many_auto_bounds_the_factorized_array(monkeypatch):
    """Above 16 placements AUTO uses the factorized evaluator unless its int64 [C, L, E] count
    array would exceed FACTORIZED_MAX_BYTES; either way (and with method="token") the integers
    are the oracle's."""
    L, E, K = B16
    m = mt.ModelSpec(L, E, K)
    N, C = 4000, 700  # short chunks
    tr = mt.generate_trace(m, 1.2, N, C, 3)
    sel, bounds = og.generate(L, E, K, 1.2, N, C, 3)
    rng = np.random.default_rng(9)
    p = rng.integers(0, 20, (L, 12)).astype(np.uint8)
    import torch
    cost = mpl.CostMatrix(torch.as_tensor(p, device="cuda"))
    pls = [mpl.Placement(random_assign(rng, L, E, 12)) for _ in range(20)]
    want = [oracle_sums(sel, p, pl.assign, bounds).tolist() for pl in pls]
    calls = []
    real = ev.score_sums_factorized
    monkeypatch.setattr(ev, "score_sums_factorized", lambda *a, **k: calls.append(1) or real(*a, **k))
    assert [r.chunk_hop_sums for r in ev.evaluate_many(tr, pls, cost)] == want
    assert calls, "factorized expected within the byte bound"
    monkeypatch.setattr(ev, "FACTORIZED_MAX_BYTES", 0)
    calls.clear()
    assert [r.chunk_hop_sums for r in ev.evaluate_many(tr, pls, cost)] == want
    assert not calls, "passes expected above the byte bound"
    assert [r.chunk_hop_sums for r in ev.evaluate_many(tr, pls, cost, method="token")] == want
