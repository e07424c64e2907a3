"""GPU parity: every device kernel against the CPU oracle, bit-exact (integers) on identical
seeded inputs, through the public API and hence the C-ABI (libmoeplace_cuda.so)."""
import numpy as np
import pytest

import moeplace.eval as ev
import moeplace.model_trace as mt
import moeplace.placement as mpl
import moeplace.solver as sv
import moeplace.topology as topo
from moeplace.errors import ConfigError, MoeplaceError, TopologyError, TraceParseError
from oracle import evaluate as oe
from oracle import gen as og
from oracle import stats as ost
from oracle import topology as ot

from helpers import B16, R1, oracle_cost, oracle_sums, random_assign, setup_topology

pytestmark = pytest.mark.gpu

SHAPES = [R1, B16, (3, 5, 2), (2, 4, 4), (1, 256, 1), (5, 200, 7)]


def _planes_tokens(tr):
    return tr.tokens()


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("s", [0.0, 1.2, 2.0])
def test_generate_matches_oracle(shape, s):
    L, E, K = shape
    N, C, seed = 1001, 7, 12345
    tr = mt.generate_trace(mt.ModelSpec(L, E, K), s, N, C, seed)
    sel, bounds = og.generate(L, E, K, s, N, C, seed)
    assert np.array_equal(tr.tokens(), sel)
    assert np.array_equal(tr.chunk_bounds, bounds)


@pytest.mark.parametrize("shape", [R1, B16])
def test_generate_shard_is_bit_identical(shape):
    L, E, K = shape
    m = mt.ModelSpec(L, E, K)
    full = mt.generate_trace(m, 1.2, 5000, 13, 99).tokens()
    for a, b in [(0, 1), (17, 1234), (4999, 5000), (2500, 5000)]:
        part = mt.generate_trace(m, 1.2, 5000, 13, 99, tok_range=(a, b))
        assert np.array_equal(part.tokens(), full[a:b])


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("s", [0.0, 1.2, 2.0])
def test_hist_matches_oracle(shape, s):
    L, E, K = shape
    N = 3001
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, s, N, 10, 7)
    sel, _ = og.generate(L, E, K, s, N, 10, 7)
    want = ost.counts(sel, E)
    f = mt.estimate_frequencies(tr, m)
    assert np.array_equal(f.counts, want)
    assert np.array_equal(f.counts, ost.counts_bincount(sel, E))
    assert np.array_equal(f.f, ost.frequencies(want, N, K))


@pytest.mark.parametrize("shape", [R1, B16, (3, 5, 2)])
def test_hist_on_unaligned_views(shape):
    """Token ranges whose byte offsets are not 16-aligned (split views) and tiny ranges."""
    L, E, K = shape
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, 1.2, 2000, 40, 3)
    sel = tr.tokens()
    for lo, hi in [(0, 1), (3, 4), (1, 39), (13, 27), (39, 40), (0, 40)]:
        v = tr.view(lo, hi)
        got = mt.estimate_frequencies(v, m).counts
        a, b = tr.chunk_bounds[lo], tr.chunk_bounds[hi]
        assert np.array_equal(got, ost.counts(sel[a:b], E)), (lo, hi)


def _assert_scores(tr, placements, costs_np, sel, bounds, t0=0):
    got = ev.score_sums(tr, placements, [c for c, _ in costs_np])
    for i, (pl, (_, p)) in enumerate(zip(placements, costs_np)):
        want = oracle_sums(sel, p, pl.assign, bounds, t0)
        assert np.array_equal(got[i], want), i


@pytest.mark.parametrize("P", [1, 3, 4, 5, 8, 9, 16, 17, 33])
def test_score_matches_oracle_R1(P):
    L, E, K = R1
    m = mt.ModelSpec(L, E, K)
    g, dist, order, attn, cost = setup_topology("FatTree", 8, 4, 8, m)
    _, p = oracle_cost(g, attn)
    assert np.array_equal(cost.numpy(), p)
    tr = mt.generate_trace(m, 1.2, 4099, 33, 5)
    sel, bounds = og.generate(L, E, K, 1.2, 4099, 33, 5)
    rng = np.random.default_rng(P)
    pls = [mpl.Placement(random_assign(rng, L, E, g.n_devices)) for _ in range(P)]
    _assert_scores(tr, pls, [(cost, p)] * P, sel, bounds)


@pytest.mark.parametrize("kind", ["FatTree", "FatTreeHier", "Dragonfly", "DragonflySparse"])
def test_score_multi_topology_16B(kind):
    """16B shape: 162 B/token is not 16-byte aligned; several topologies in one batch."""
    L, E, K = B16
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, 1.2, 2777, 11, 8)
    sel, bounds = og.generate(L, E, K, 1.2, 2777, 11, 8)
    costs, pls = [], []
    for i, kd in enumerate([kind, "FatTree", "Dragonfly"]):
        g, dist, order, attn, cost = setup_topology(kd, 4, 2, 4, m)
        _, p = oracle_cost(g, attn)
        for j in range(3):
            pls.append(mpl.Placement(random_assign(np.random.default_rng(10 * i + j), L, E, g.n_devices)))
            costs.append((cost, p))
    _assert_scores(tr, pls, costs, sel, bounds)


def test_score_views_and_empty_chunks():
    L, E, K = B16
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, 2.0, 90, 150, 1)  # N < C: many empty chunks
    sel, bounds = og.generate(L, E, K, 2.0, 90, 150, 1)
    g, dist, order, attn, cost = setup_topology("Dragonfly", 8, 1, 4, m)
    _, p = oracle_cost(g, attn)
    pl = mpl.Placement(random_assign(np.random.default_rng(0), L, E, g.n_devices))
    rep = ev.evaluate(tr, pl, cost)
    want = oracle_sums(sel, p, pl.assign, bounds)
    assert rep.chunk_hop_sums == want.tolist()
    r = oe.report(want, np.diff(bounds))
    assert rep.mean_hops_per_token == r["mean"] and rep.std_hops == r["std"]
    assert rep.empty_chunks == r["empty_chunks"] == 60
    train, test = mt.split_trace(tr, 100, 50)
    rt = ev.evaluate(test, pl, cost)
    assert rt.chunk_hop_sums == want[100:150].tolist()


@pytest.mark.parametrize("maxp_kind", ["small", "mid", "large"])
def test_score_widening_paths(maxp_kind):
    """u8-lane widening intervals (max_p <= 15, <= 63, <= 255) give identical sums."""
    L, E, K = (4, 64, 8)
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, 1.2, 3333, 5, 2)
    sel, bounds = og.generate(L, E, K, 1.2, 3333, 5, 2)
    hi = {"small": 15, "mid": 63, "large": 255}[maxp_kind]
    rng = np.random.default_rng(hi)
    S = 16
    p = rng.integers(0, hi + 1, size=(L, S)).astype(np.uint8)
    p[0, 0] = hi
    import torch
    cost = mpl.CostMatrix(torch.as_tensor(p, device="cuda"))
    pls = [mpl.Placement(random_assign(rng, L, E, S)) for _ in range(6)]
    _assert_scores(tr, pls, [(cost, p)] * 6, sel, bounds)


def test_fused_hist_score_matches():
    L, E, K = R1
    m = mt.ModelSpec(L, E, K)
    g, dist, order, attn, cost = setup_topology("DragonflySparse", 16, 4, 4, m)
    _, p = oracle_cost(g, attn)
    tr = mt.generate_trace(m, 1.2, 3001, 20, 4)
    sel, bounds = og.generate(L, E, K, 1.2, 3001, 20, 4)
    train, _ = mt.split_trace(tr, 13, 7)
    rng = np.random.default_rng(1)
    pls = [mpl.Placement(random_assign(rng, L, E, g.n_devices)) for _ in range(4)]
    freq, reps = ev.evaluate_with_stats(train, pls, cost)
    b = bounds[13]
    assert np.array_equal(freq.counts, ost.counts(sel[:b], E))
    for pl, rep in zip(pls, reps):
        assert rep.chunk_hop_sums == oracle_sums(sel[:b], p, pl.assign, bounds[:14]).tolist()


@pytest.mark.parametrize("kind,leaves,spl,gps", [
    ("FatTree", 16, 4, 4), ("FatTreeHier", 16, 4, 4), ("Dragonfly", 16, 4, 4), ("DragonflySparse", 16, 4, 4),
    ("DragonflySparse", 64, 1, 1), ("Dragonfly", 64, 1, 1), ("FatTree", 8, 4, 8), ("DragonflyPlus", 16, 4, 4),
    ("SlimFly", 18, 1, 2), ("SlimFly", 50, 1, 1), ("FatTreeHier", 3, 2, 1), ("DragonflySparse", 1, 1, 4)])
def test_apsp_matches_bfs_oracle(kind, leaves, spl, gps):
    import networkx as nx
    g = topo.build_topology(topo.TopologySpec(kind, leaves, spl, gps))
    d = topo.all_pairs_hops(g)
    want = ot.server_hops(g.n_nodes, g.links.tolist(), g.n_servers)
    assert np.array_equal(d.server_numpy(), want)
    G = nx.Graph()
    G.add_nodes_from(range(g.n_nodes))
    G.add_edges_from(g.links.tolist())
    sp = dict(nx.all_pairs_shortest_path_length(G))
    assert all(want[a, b] == sp[a][b] for a in range(g.n_servers) for b in range(g.n_servers))
    D = d.numpy()
    assert np.array_equal(D, ot.device_hops(want, g.device_server))
    assert (D == D.T).all() and (np.diag(D) == 0).all()


def test_apsp_disconnected_raises():
    g = topo.build_topology(topo.TopologySpec("FatTree", 2, 1, 1, {"spines": 1}))
    g.links = g.links[:-1]  # drop a leaf-spine link
    with pytest.raises(TopologyError):
        topo.all_pairs_hops(g)


def test_cost_matrix_matches_oracle():
    for kind in ("FatTree", "FatTreeHier", "Dragonfly", "DragonflySparse"):
        m = mt.ModelSpec(58, 256, 8)
        g, dist, order, attn, cost = setup_topology(kind, 16, 4, 4, m)
        _, p = oracle_cost(g, attn)
        assert np.array_equal(cost.numpy(), p)


@pytest.mark.parametrize("uniform", [True, False])
def test_coefficients_bit_exact(uniform):
    L, E, K = B16
    m = mt.ModelSpec(L, E, K)
    g, dist, order, attn, cost = setup_topology("Dragonfly", 2, 2, 8, m)
    tr = mt.generate_trace(m, 1.2, 5000, 10, 3)
    c = mpl.Constraints(54, 2)
    if uniform:
        inst = sv.build_instance(cost, sv.UniformFrequencies(E), c)
        f = np.full((L, E), 1.0 / E)
    else:
        freq = mt.estimate_frequencies(tr, m)
        inst = sv.build_instance(cost, freq, c)
        f = freq.counts / (K * 5000)
    w, wi = ot.coefficients(f, cost.numpy())
    assert np.array_equal(inst.w_numpy(), w)  # bit-identical float64
    assert np.array_equal(inst.w_int_numpy(), wi)


def test_comm_map_matches_oracle():
    L, E, K = B16
    m = mt.ModelSpec(L, E, K)
    g, dist, order, attn, cost = setup_topology("FatTreeHier", 8, 2, 2, m)
    tr = mt.generate_trace(m, 1.2, 2000, 10, 3)
    pl = mpl.place_greedy(m, attn, cost, mpl.Constraints(64, 2))
    cm = ev.communication_map(tr, pl, cost)
    cnt = ost.counts(tr.tokens(), E)
    sym, raw = oe.comm_map(cnt, pl.assign, g.device_server, dist.server_numpy(), attn.dispatch, attn.collect, 2000)
    assert np.array_equal(cm.raw, raw)
    assert np.array_equal(cm.traffic, sym)
    rep = ev.evaluate(tr, pl, cost)
    assert abs(cm.traffic.sum() - rep.mean_hops_per_token) <= 1e-9 * rep.mean_hops_per_token
    assert np.allclose(cm.traffic, cm.traffic.T) and (np.diag(cm.traffic) == 0).all()


def test_golden_fixture(golden_dir):
    z = np.load(golden_dir / "oracle_small.npz")
    L, E, K, N, C = (int(z[k]) for k in ("L", "E", "K", "N", "C"))
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, float(z["zipf_s"]), N, C, int(z["seed"]))
    assert np.array_equal(tr.tokens(), z["sel"])
    assert np.array_equal(mt.estimate_frequencies(tr, m).counts, z["counts"])
    import torch
    cost = mpl.CostMatrix(torch.as_tensor(z["p"].astype(np.uint8), device="cuda"))
    rep = ev.evaluate(tr, mpl.Placement(z["assign"]), cost)
    assert rep.chunk_hop_sums == z["sums"].tolist()


def test_token_hops_spec_examples():
    import torch
    p = mpl.CostMatrix(torch.as_tensor(np.array([[4, 2]], np.uint8), device="cuda"))
    assert ev.token_hops([[0, 1]], mpl.Placement(np.array([[0, 1]])), p) == 6
    p0 = mpl.CostMatrix(torch.as_tensor(np.array([[0, 4, 4]], np.uint8), device="cuda"))
    assert ev.token_hops([[0, 2]], mpl.Placement(np.array([[0, 0, 0]])), p0) == 0


def test_data_errors_are_reported():
    m = mt.ModelSpec(2, 4, 2)
    sel = np.array([[[0, 1], [2, 3]], [[1, 1], [0, 2]]], dtype=np.uint8)  # token 1 layer 0 repeats
    tr = mt.ActivationTrace.from_tokens(m, sel)
    with pytest.raises(MoeplaceError):
        mt.estimate_frequencies(tr, m)
    bad = np.array([[[0, 9], [2, 3]]], dtype=np.uint8)
    import torch
    tr2 = mt.ActivationTrace(m, torch.from_numpy(bad), 0, 1, np.zeros(1, np.int64), np.array([0, 1], np.int64),
                             layout="tokens")  # token-major host trace: validated slice by slice on the device
    with pytest.raises(MoeplaceError):
        mt.estimate_frequencies(tr2, m)
    with pytest.raises(MoeplaceError):
        mt.estimate_frequencies(tr.view(0, 0), m)


def test_parse_file_errors_carry_line_numbers(tmp_path):
    m = mt.ModelSpec(2, 4, 2)
    tr = mt.generate_trace(m, 1.2, 5, 2, 1)
    f = tmp_path / "t.txt"
    mt.write_trace(tr, f)
    lines = f.read_text().splitlines()
    lines[3] = lines[3].replace("layer1:", "layer1:4,")  # wrong count at line 4
    f.write_text("\n".join(lines) + "\n")
    with pytest.raises(TraceParseError) as ei:
        mt.parse_trace(f)
    assert ei.value.line_no == 4


def test_large_trace_properties():
    """At BASELINE's full R1 size (10M tokens): size-independent properties + a sampled oracle
    check on a shard regenerated independently on the CPU."""
    L, E, K = R1
    m = mt.ModelSpec(L, E, K)
    N, C = 10_000_000, 150
    tr = mt.generate_trace(m, 1.2, N, C, 0)
    cnt = mt.estimate_frequencies(tr, m).counts
    assert (cnt.sum(axis=1) == N * K).all()
    import torch
    S = 64
    q = np.full((L, S), 3, np.uint8)
    cost = mpl.CostMatrix(torch.as_tensor(q, device="cuda"))
    rng = np.random.default_rng(0)
    pl = mpl.Placement(random_assign(rng, L, E, S))
    rep = ev.evaluate(tr, pl, cost)
    assert rep.hop_sum == 3 * N * L * K  # constant p -> every pick costs 3
    # linearity: score(p1) + score(p2) == score(p1 + p2)
    p1 = rng.integers(0, 8, (L, S)).astype(np.uint8)
    p2 = rng.integers(0, 8, (L, S)).astype(np.uint8)
    c1, c2, c12 = (mpl.CostMatrix(torch.as_tensor(x, device="cuda")) for x in (p1, p2, p1 + p2))
    s = ev.score_sums(tr, [pl, pl, pl], [c1, c2, c12])
    assert np.array_equal(s[0] + s[1], s[2])
    # identity with the histogram: sum_{l,e} count * pe == total hops
    pe = oe.pe_table(p1, pl.assign)
    assert int((cnt * pe).sum()) == int(s[0].sum())
    # sampled oracle check: tokens [a, b) regenerated on the CPU
    a, b = 4_321_000, 4_331_000
    sel, bounds = og.generate(L, E, K, 1.2, N, C, 0, tok_range=(a, b))
    sh = mt.generate_trace(m, 1.2, N, C, 0, tok_range=(a, b))
    assert np.array_equal(sh.tokens(), sel)
    got = ev.score_sums(sh, [pl], c1)[0]
    assert np.array_equal(got, oe.chunk_sums(sel, pe, bounds, a))


def test_host_streaming_matches_device(monkeypatch):
    """The end-to-end path (pinned host planes streamed through device slices) gives the same
    integers as the device-resident path, with slices that cut through chunks."""
    import moeplace.model_trace as mtm
    monkeypatch.setattr(mtm, "STREAM_BLOCK_TOKENS", 777)
    L, E, K = B16
    m = mt.ModelSpec(L, E, K)
    g, dist, order, attn, cost = setup_topology("FatTree", 2, 2, 8, m)
    tr = mt.generate_trace(m, 1.2, 5000, 9, 21)
    rng = np.random.default_rng(3)
    pls = [mpl.Placement(random_assign(rng, L, E, g.n_devices)) for _ in range(6)]
    want = ev.score_sums(tr, pls, cost)
    f_dev, r_dev = ev.evaluate_with_stats(tr, pls[:4], cost)
    host = tr.to_host(pin=True)
    assert not host.planes.is_cuda
    assert np.array_equal(ev.score_sums(host, pls, cost), want)
    f_h, r_h = ev.evaluate_with_stats(host, pls[:4], cost)
    assert np.array_equal(f_h.counts, f_dev.counts)
    assert [r.chunk_hop_sums for r in r_h] == [r.chunk_hop_sums for r in r_dev]
    assert np.array_equal(mt.estimate_frequencies(host, m).counts, f_dev.counts)
    assert not host.planes.is_cuda  # streamed, not cached on the device


@pytest.mark.parametrize("shape", [R1, B16, (3, 5, 2)])
def test_token_major_host_streaming_matches_device(monkeypatch, shape):
    """SPEC-shaped end-to-end input: token-major [N, L, K] selections in pinned host memory,
    streamed slice by slice and transposed on the device (mp_tokens_to_planes_u8; K = 8 takes the
    tiled u64 transpose), give the device-resident integers -- slices cut through chunks, views
    start mid-slice, per-token hops land at the right offsets."""
    import moeplace.model_trace as mtm
    monkeypatch.setattr(mtm, "STREAM_BLOCK_TOKENS", 1000)
    L, E, K = shape
    m = mt.ModelSpec(L, E, K)
    g, dist, order, attn, cost = setup_topology("FatTree", 2, 2, 8, m)
    tr = mt.generate_trace(m, 1.2, 4321, 9, 21)
    rng = np.random.default_rng(3)
    pls = [mpl.Placement(random_assign(rng, L, E, g.n_devices)) for _ in range(5)]
    host = mt.ActivationTrace.from_host_tokens(m, tr.tokens(), tr.chunk_bounds)
    assert host.layout == "tokens" and host.planes.is_pinned()
    assert np.array_equal(host.tokens(), tr.tokens())
    assert np.array_equal(ev.score_sums(host, pls, cost), ev.score_sums(tr, pls, cost))
    f_h, r_h = ev.evaluate_with_stats(host, pls[:4], cost)
    f_d, r_d = ev.evaluate_with_stats(tr, pls[:4], cost)
    assert np.array_equal(f_h.counts, f_d.counts)
    assert [r.chunk_hop_sums for r in r_h] == [r.chunk_hop_sums for r in r_d]
    v_h, v_d = host.view(2, 7), tr.view(2, 7)
    assert np.array_equal(ev.score_sums(v_h, pls, cost), ev.score_sums(v_d, pls, cost))
    assert np.array_equal(ev.token_hops_all(v_h, pls[:2], cost), ev.token_hops_all(v_d, pls[:2], cost))
    assert np.array_equal(v_h.device_planes()[:, :v_h.n_tokens * K].cpu().numpy(),
                          v_d.planes[:, v_d.tok_begin * K:v_d.tok_end * K].cpu().numpy())
    # router ids on the device: the same transpose kernel
    import torch
    r = mt.ActivationTrace.from_router_topk(m, torch.as_tensor(tr.tokens(), device="cuda").long(), tr.chunk_bounds)
    assert np.array_equal(r.tokens(), tr.tokens())
    # invalid ids in a token-major host trace are caught while streaming
    bad = tr.tokens()
    bad[1234, L - 1, 0] = bad[1234, L - 1, K - 1] if K > 1 else E
    hb = mt.ActivationTrace.from_host_tokens(m, bad, tr.chunk_bounds)
    with pytest.raises(MoeplaceError):
        mt.estimate_frequencies(hb, m)


@pytest.mark.parametrize("shape,kind,size", [
    (R1, "FatTree", (4, 2, 4)), (B16, "Dragonfly", (4, 2, 4)), ((3, 16, 5), "DragonflySparse", (4, 2, 4)),
    # K = 8 general path: pe bytes up to 36 in some layers (fast and general layers mixed), and
    # 130 servers (ids >= 128)
    (R1, "DragonflySparse", (64, 1, 1)), (R1, "FatTree", (65, 2, 1)),
    # one-hot path (every server id < 32, costs <= 15): config 2's 32-server FatTree; 32 servers of a
    # sparse dragonfly whose larger costs send some layers back to the pairwise path
    (R1, "FatTree", (8, 4, 8)), (R1, "DragonflySparse", (32, 1, 1))])
def test_dedup_matches_oracle(shape, kind, size):
    """Extension A17: unique destination servers and deduplicated hops, bit-exact vs the oracle;
    the SPEC hop sums produced alongside equal mp_score_u8's."""
    L, E, K = shape
    m = mt.ModelSpec(L, E, K)
    g, dist, order, attn, cost = setup_topology(kind, *size, m)
    _, p = oracle_cost(g, attn)
    tr = mt.generate_trace(m, 1.2, 2345, 9, 6)
    sel, bounds = og.generate(L, E, K, 1.2, 2345, 9, 6)
    rng = np.random.default_rng(2)
    pls = [mpl.Placement(random_assign(rng, L, E, g.n_devices)) for _ in range(6)]
    reps = ev.evaluate_dedup(tr, pls, cost)
    spec = ev.score_sums(tr, pls, cost)
    src = g.device_server[attn.dispatch]
    for i, (pl, rep) in enumerate(zip(pls, reps)):
        pe = oe.pe_table(p, pl.assign)
        h, u, d = oe.dedup_sums(sel, pe, g.device_server[pl.assign], src, bounds)
        assert rep.spec.chunk_hop_sums == h.tolist() == spec[i].tolist()
        assert rep.chunk_uniq_sums == u.tolist()
        assert rep.chunk_dedup_sums == d.tolist()
        assert (d <= h).all()


def _write_lines(path, lines, trailing="\n"):
    path.write_text("\n".join(lines) + trailing)


@pytest.mark.parametrize("lines,line_no", [
    (["#moeplace-trace v1 L=2 E=4 K=2", "0\tlayer0:0,1\tlayer1:2,3", "0\tlayer0:0,4\tlayer1:2,3"], 3),
    (["#moeplace-trace v1 L=2 E=4 K=2", "0\tlayer0:0,1"], 2),
    (["#moeplace-trace v1 L=2 E=4 K=2", "0\tlayer0:0,1\tlayer1:2,2"], 2),
    (["#moeplace-trace v1 L=2 E=4 K=2", "0\tlayer0:0,1\tlayer1:2,3", "1\tlayer1:0,1\tlayer0:2,3"], 3),
    (["#moeplace-trace v1 L=2 E=4 K=2", "0\tlayer0:0,1,2\tlayer1:2,3"], 2),
    (["#moeplace-trace v1 L=2 E=4 K=2", "x\tlayer0:0,1\tlayer1:2,3"], 2),
    (["#moeplace-trace v1 L=2 E=4 K=2", "0\tlayer0:0,1\tlayer1:2,3", ""], 3),
    (["garbage"], 1),
])
def test_device_parser_errors_match_oracle(tmp_path, lines, line_no):
    from oracle.textio import TextParseError, parse_text
    f = tmp_path / "t.txt"
    _write_lines(f, lines)
    with pytest.raises(TextParseError) as e:
        parse_text(f)
    assert e.value.line_no == line_no
    with pytest.raises(TraceParseError) as e:
        mt.parse_trace(f)
    assert e.value.line_no == line_no


def test_device_parser_roundtrip_and_regroup(tmp_path):
    m = mt.ModelSpec(27, 64, 6)
    tr = mt.generate_trace(m, 1.2, 3001, 17, 5)
    f = tmp_path / "t.txt"
    mt.write_trace(tr, f)
    from oracle.textio import parse_text, regroup
    d = mt.parse_trace(f)  # device engine
    _, hsel, hcid = parse_text(f)
    assert d.planes.is_cuda
    assert np.array_equal(d.tokens(), tr.tokens()) and np.array_equal(hsel, tr.tokens())
    assert np.array_equal(d.chunk_bounds, tr.chunk_bounds) and np.array_equal(d.chunk_ids, tr.chunk_ids)
    g = tmp_path / "u.txt"
    mt.write_trace(d, g)
    assert g.read_bytes() == f.read_bytes()
    # prefix-less fields, CRLF, no trailing newline, interleaved chunk ids -> stable regroup
    lines = ["#moeplace-trace v1 L=2 E=5 K=2", "7\t0:0,1\t1:2,3\r", "3\tlayer0:4,1\tlayer1:0,3", "7\tlayer0:2,1\t1:2,4"]
    _write_lines(tmp_path / "v.txt", lines, trailing="")
    a = mt.parse_trace(tmp_path / "v.txt")
    bsel, _, _ = regroup(*parse_text(tmp_path / "v.txt")[1:])
    assert np.array_equal(a.tokens(), bsel)
    assert a.chunk_ids.tolist() == [3, 7] and a.chunk_bounds.tolist() == [0, 1, 3]
    assert a.tokens()[:, 0, :].tolist() == [[4, 1], [0, 1], [2, 1]]


def test_device_parser_R1_scale(tmp_path):
    """A 20k-token R1 file through the device parser equals the generator's planes, and the
    stats/score computed from it equal the oracle's."""
    L, E, K = R1
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, 1.2, 20000, 30, 9)
    f = tmp_path / "r1.txt"
    mt.write_trace(tr, f)
    d = mt.parse_trace(f)
    assert np.array_equal(d.tokens(), tr.tokens())
    sel, _ = og.generate(L, E, K, 1.2, 20000, 30, 9)
    assert np.array_equal(mt.estimate_frequencies(d, m).counts, ost.counts(sel, E))


@pytest.mark.parametrize("shape,kind,maxp", [(R1, "FatTree", None), (B16, "DragonflySparse", None),
                                             ((5, 32, 8), None, 200), ((3, 64, 3), None, 100),
                                             # K = 8 accumulation widths: u8 per token (<= 31), per 4 (<= 63)
                                             ((4, 64, 8), None, 31), ((4, 64, 8), None, 50), ((4, 64, 8), None, 63)])
def test_token_hops_all_matches_oracle(shape, kind, maxp):
    """Per-token hops of every token (token-tiled kernel) == the oracle's per-token sums; chunk
    sums of them == the streaming scorer's."""
    import torch
    L, E, K = shape
    m = mt.ModelSpec(L, E, K)
    N = 9000
    tr = mt.generate_trace(m, 1.2, N, 13, 4)
    sel, bounds = og.generate(L, E, K, 1.2, N, 13, 4)
    rng = np.random.default_rng(5)
    if kind:
        g, dist, order, attn, cost = setup_topology(kind, 4, 2, 4, m)
        p = cost.numpy()
        S = g.n_devices
    else:
        S = 16
        p = rng.integers(0, maxp + 1, (L, S)).astype(np.uint8)
        p[0, 0] = maxp  # pin the accumulation-width boundary
        cost = mpl.CostMatrix(torch.as_tensor(p, device="cuda"))
    pls = [mpl.Placement(random_assign(rng, L, E, S)) for _ in range(6)]
    got = ev.token_hops_all(tr, pls, cost)
    sums = ev.score_sums(tr, pls, cost)
    for i, pl in enumerate(pls):
        want = oe.per_token_hops(sel, oe.pe_table(p, pl.assign))
        assert np.array_equal(got[i], want)
        assert np.array_equal(np.add.reduceat(got[i], bounds[:-1]) if (np.diff(bounds) > 0).all() else sums[i],
                              sums[i])
    v = tr.view(2, 9)
    gv = ev.token_hops_all(v, pls[:1], cost)[0]
    assert np.array_equal(gv, got[0][bounds[2]:bounds[9]])
    assert ev.hop_distribution(tr, pls[0], cost).sum() == N


def test_token_hops_all_multi_tile_ranges():
    """Per-CTA token ranges of several 4096-token tiles (the TMA ring walks tile x layer steps across
    tile ends), an odd token count and a view starting on an odd token (slices 8 bytes into a
    16-byte line) == the oracle."""
    import torch
    L, E, K = 3, 256, 8
    m = mt.ModelSpec(L, E, K)
    N = 1_300_001
    tr = mt.generate_trace(m, 1.2, N, 7, 11)
    sel, bounds = og.generate(L, E, K, 1.2, N, 7, 11)
    rng = np.random.default_rng(8)
    p = rng.integers(0, 32, (L, 16)).astype(np.uint8)
    cost = mpl.CostMatrix(torch.as_tensor(p, device="cuda"))
    pls = [mpl.Placement(random_assign(rng, L, E, 16)) for _ in range(2)]
    got = ev.token_hops_all(tr, pls, cost)
    for i, pl in enumerate(pls):
        assert np.array_equal(got[i], oe.per_token_hops(sel, oe.pe_table(p, pl.assign)))
    odd = next(c for c in range(1, 7) if bounds[c] % 2 == 1) if any(b % 2 for b in bounds[1:7]) else 1
    v = tr.view(odd, 7)
    gv = ev.token_hops_all(v, pls[:1], cost)[0]
    assert np.array_equal(gv, got[0][bounds[odd]:bounds[7]])


@pytest.mark.parametrize("shape", [R1, B16, (3, 5, 2)])
def test_factorized_evaluator_matches_gather(shape):
    """per-chunk histograms + exact contraction == per-token gather, bit for bit, for
    many placements over several topologies; per-chunk counts == oracle per chunk."""
    L, E, K = shape
    m = mt.ModelSpec(L, E, K)
    N, C = 5003, 23
    tr = mt.generate_trace(m, 1.2, N, C, 8)
    sel, bounds = og.generate(L, E, K, 1.2, N, C, 8)
    cc = mt.chunk_counts(tr).cpu().numpy()
    for c in range(C):
        assert np.array_equal(cc[c], ost.counts(sel[bounds[c]:bounds[c + 1]], E)), c
    costs, pls = [], []
    for i, kind in enumerate(["FatTree", "Dragonfly", "DragonflySparse"]):
        g, dist, order, attn, cost = setup_topology(kind, 4, 2, 2, m)
        for j in range(7):
            pls.append(mpl.Placement(random_assign(np.random.default_rng(31 * i + j), L, E, g.n_devices)))
            costs.append(cost)
    a = ev.score_sums(tr, pls, costs)
    b = ev.score_sums_factorized(tr, pls, costs)
    c2 = ev.score_sums_factorized(tr, pls, costs, contraction="cuda")
    assert np.array_equal(a, b) and np.array_equal(a, c2)
    ra = ev.evaluate_many(tr.view(3, 20), pls[:5], costs[:5])
    rb = ev.evaluate_many(tr.view(3, 20), pls[:5], costs[:5], method="factorized")
    assert [r.chunk_hop_sums for r in ra] == [r.chunk_hop_sums for r in rb]


@pytest.mark.parametrize("P,LE,C,pe_hi", [(37, 1000, 11, 256), (37, 1000, 11, 128), (64, 1024, 8, 256),
                                          (64, 1024, 13, 100), (4096, 14848, 150, 13)])
def test_contract_tc_digit_paths(P, LE, C, pe_hi):
    """Exact tensor-core contraction with multi-digit operands (pe up to 255, counts up to 2^20),
    padded and GEMM-aligned (no-copy) operand shapes."""
    import torch
    rng = np.random.default_rng(P + C)
    pe = torch.as_tensor(rng.integers(0, pe_hi, (P, LE)).astype(np.uint8), device="cuda")
    cnt = torch.as_tensor(rng.integers(0, 2 ** 20, (C, LE)), device="cuda")
    got = ev.contract_tc(cnt, pe).cpu().numpy()
    want = pe.cpu().numpy().astype(np.int64) @ cnt.cpu().numpy().T
    assert np.array_equal(got, want)
    # stated operand bounds (no device reductions) give the same integers
    bounded = ev.contract_tc(cnt, pe, max_count=2 ** 20 - 1, max_pe=pe_hi - 1).cpu().numpy()
    assert np.array_equal(bounded, want)


def test_contract_tc_count_above_the_stated_bound_raises():
    import torch
    from moeplace.errors import MoeplaceError
    pe = torch.ones((40, 64), dtype=torch.uint8, device="cuda")
    cnt = torch.full((9, 64), 300, dtype=torch.int64, device="cuda")
    assert ev.contract_tc(cnt, pe, max_count=300).sum().item() == 40 * 9 * 64 * 300
    with pytest.raises(MoeplaceError):
        ev.contract_tc(cnt, pe, max_count=100)  # one 8-bit digit cannot hold 300: raised, not truncated


@pytest.mark.parametrize("shape", [R1, B16, (2, 4, 1), (1, 256, 3)])
def test_device_writer_matches_oracle_writer(tmp_path, shape):
    from oracle.textio import write_text
    L, E, K = shape
    m = mt.ModelSpec(L, E, K)
    tr = mt.generate_trace(m, 1.2, 1234, 11, 3)
    mt.write_trace(tr, tmp_path / "d.txt")
    write_text(tmp_path / "h.txt", (L, E, K), tr.tokens(), tr.token_chunk_ids())
    assert (tmp_path / "d.txt").read_bytes() == (tmp_path / "h.txt").read_bytes()
    v = tr.view(2, 7)
    mt.write_trace(v, tmp_path / "dv.txt")
    write_text(tmp_path / "hv.txt", (L, E, K), v.tokens(), v.token_chunk_ids())
    assert (tmp_path / "dv.txt").read_bytes() == (tmp_path / "hv.txt").read_bytes()
    # a host-resident trace (pinned planes or token-major) is written through the device too
    mt.write_trace(v.to_host(pin=True), tmp_path / "dh.txt")
    mt.write_trace(tr.to_host(pin=True, layout="tokens").view(2, 7), tmp_path / "dt.txt")
    assert (tmp_path / "dh.txt").read_bytes() == (tmp_path / "dt.txt").read_bytes() == (tmp_path / "hv.txt").read_bytes()
    back = mt.parse_trace(tmp_path / "d.txt")
    assert np.array_equal(back.tokens(), tr.tokens())


@pytest.mark.parametrize("shape", [(3, 64, 16), (2, 256, 32), (4, 1, 1), (1, 33, 33)])
def test_wide_k_and_degenerate_shapes(tmp_path, shape):
    """K = 16 / 32 (generic generator, byte paths), E = 1, K = E: generator, histogram, score,
    fused pass, dedup, per-token hops, parser and writer all agree with the oracle."""
    import torch
    L, E, K = shape
    m = mt.ModelSpec(L, E, K)
    N, C = 777, 5
    tr = mt.generate_trace(m, 1.2, N, C, 2)
    sel, bounds = og.generate(L, E, K, 1.2, N, C, 2)
    assert np.array_equal(tr.tokens(), sel)
    assert np.array_equal(mt.estimate_frequencies(tr, m).counts, ost.counts(sel, E))
    rng = np.random.default_rng(9)
    S = 8
    p = rng.integers(0, 7, (L, S)).astype(np.uint8)
    cost = mpl.CostMatrix(torch.as_tensor(p, device="cuda"))
    pls = [mpl.Placement(random_assign(rng, L, E, S)) for _ in range(5)]
    got = ev.score_sums(tr, pls, cost)
    for i, pl in enumerate(pls):
        assert np.array_equal(got[i], oracle_sums(sel, p, pl.assign, bounds))
    f, reps = ev.evaluate_with_stats(tr, pls[:4], cost)
    assert np.array_equal(f.counts, ost.counts(sel, E))
    assert [r.chunk_hop_sums for r in reps] == [got[i].tolist() for i in range(4)]
    th = ev.token_hops_all(tr, pls[:2], cost)
    for i in range(2):
        assert np.array_equal(th[i], oe.per_token_hops(sel, oe.pe_table(p, pls[i].assign)))
    assert np.array_equal(ev.score_sums_factorized(tr, pls, cost), got)
    mt.write_trace(tr, tmp_path / "t.txt")
    assert np.array_equal(mt.parse_trace(tmp_path / "t.txt").tokens(), sel)


@pytest.mark.parametrize("shape", [R1, B16, (3, 64, 5)])
def test_poisoned_padding_is_never_read(shape):
    """Guard band (compute-sanitizer is unavailable on this pool): plane bytes beyond the valid
    tokens are filled with an out-of-range id; every kernel must ignore them (the histogram
    range check would raise, sums would change)."""
    import torch
    L, E, K = shape
    m = mt.ModelSpec(L, E, K)
    N, C = 2001, 9
    tr = mt.generate_trace(m, 1.2, N, C, 4)
    stride = ((N * K + 15) // 16) * 16 + 4096
    planes = torch.full((L, stride), 255 if E < 256 else 0, dtype=torch.uint8, device="cuda")
    planes[:, :N * K] = tr.planes[:, :N * K]
    poisoned = mt.ActivationTrace(m, planes, 0, N, tr.chunk_ids.copy(), tr.chunk_bounds.copy(), _validated=True)
    sel, bounds = og.generate(L, E, K, 1.2, N, C, 4)
    assert np.array_equal(mt.estimate_frequencies(poisoned, m).counts, ost.counts(sel, E))
    rng = np.random.default_rng(1)
    S = 8
    p = rng.integers(1, 9, (L, S)).astype(np.uint8)
    cost = mpl.CostMatrix(torch.as_tensor(p, device="cuda"))
    pls = [mpl.Placement(random_assign(rng, L, E, S)) for _ in range(9)]
    want = np.stack([oracle_sums(sel, p, pl.assign, bounds) for pl in pls])
    assert np.array_equal(ev.score_sums(poisoned, pls, cost), want)
    assert np.array_equal(ev.score_sums_factorized(poisoned, pls, cost), want)
    f, reps = ev.evaluate_with_stats(poisoned, pls[:4], cost)
    assert [r.chunk_hop_sums for r in reps] == want[:4].tolist()
    th = ev.token_hops_all(poisoned, pls[:1], cost)[0]
    assert np.array_equal(th, oe.per_token_hops(sel, oe.pe_table(p, pls[0].assign)))


def test_from_router_topk_device_ingestion():
    import torch
    m = mt.ModelSpec(5, 64, 6)
    sel, bounds = og.generate(5, 64, 6, 1.2, 3000, 7, 5)
    ids = torch.as_tensor(sel.astype(np.int64), device="cuda")
    tr = mt.ActivationTrace.from_router_topk(m, ids, bounds)
    assert np.array_equal(tr.tokens(), sel)
    assert np.array_equal(mt.estimate_frequencies(tr, m).counts, ost.counts(sel, 64))
    bad = ids.clone()
    bad[7, 2, 1] = bad[7, 2, 0]  # duplicate id in one record
    with pytest.raises(MoeplaceError):
        mt.ActivationTrace.from_router_topk(m, bad, bounds)
    with pytest.raises(MoeplaceError):
        mt.ActivationTrace.from_router_topk(m, ids + 64, bounds)


def test_binary_sidecar_roundtrip(tmp_path):
    m = mt.ModelSpec(27, 64, 6)
    tr = mt.generate_trace(m, 1.2, 5001, 13, 2)
    v = tr.view(2, 11)
    mt.write_trace_binary(v, tmp_path / "t.mptrace")
    for dev in ("pinned", "cuda"):
        b = mt.read_trace_binary(tmp_path / "t.mptrace", device=dev)
        assert np.array_equal(b.tokens(), v.tokens())
        assert np.array_equal(b.chunk_ids, v.chunk_ids)
        assert np.array_equal(b.chunk_bounds, v.chunk_bounds - v.tok_begin)
        assert np.array_equal(mt.estimate_frequencies(b, m).counts, mt.estimate_frequencies(v, m).counts)
    (tmp_path / "bad").write_bytes(b"NOTATRACE" * 4)
    with pytest.raises(TraceParseError):
        mt.read_trace_binary(tmp_path / "bad")


def test_exact_integer_coefficients_same_optimum():
    """exact count*p flow costs give the same optimal objective as the 1e9-scaled
    SPEC costs (positive scaling) — and are exactly counts * p."""
    L, E, K = B16
    m = mt.ModelSpec(L, E, K)
    g, dist, order, attn, cost = setup_topology("Dragonfly", 2, 2, 8, m)
    tr = mt.generate_trace(m, 1.2, 20000, 10, 3)
    freq = mt.estimate_frequencies(tr, m)
    c = mpl.Constraints(54, 2)
    a = sv.build_instance(cost, freq, c)
    b = sv.build_instance(cost, freq, c, exact=True)
    assert np.array_equal(b.w_int_numpy(), freq.counts[:, :, None] * cost.numpy().astype(np.int64)[:, None, :])
    pa, oa = sv.solve_exact(a)
    pb, ob = sv.solve_exact(b)
    assert abs(oa - ob) <= 1e-12 * max(1.0, oa)
    assert ev.objective_value(pa, freq, cost) == pytest.approx(ev.objective_value(pb, freq, cost), rel=1e-12)


def test_single_chunk_std_zero_and_p_sweep():
    """C = 1 gives std = 0 exactly; P in {1, 4, 16} on E = 64 / 256."""
    import torch
    for (L, E, K) in [(4, 64, 6), (3, 256, 8)]:
        m = mt.ModelSpec(L, E, K)
        tr = mt.generate_trace(m, 1.2, 1237, 1, 2)
        rng = np.random.default_rng(E)
        p = rng.integers(0, 9, (L, 8)).astype(np.uint8)
        cost = mpl.CostMatrix(torch.as_tensor(p, device="cuda"))
        for P in (1, 4, 16):
            pls = [mpl.Placement(random_assign(rng, L, E, 8)) for _ in range(P)]
            reps = ev.evaluate_many(tr, pls, cost)
            assert all(r.std_hops == 0.0 and r.n_chunks == 1 for r in reps)
