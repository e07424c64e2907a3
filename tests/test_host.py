"""Host-side logic of the moeplace API (no GPU): topology wiring, locality ordering, attention
default, placers, validation, the native min-cost-flow solver vs brute force and HiGHS, file
formats, config handling and the error classes."""
import json

import numpy as np
import pytest

import moeplace.cli as cli
import moeplace.model_trace as mt
import moeplace.placement as mpl
import moeplace.solver as sv
import moeplace.topology as topo
from moeplace.errors import (ConfigError, InfeasibleError, MoeplaceError, TopologyError, TraceParseError,
                             exit_code)
from oracle import topology as ot


class HostDist:
    """A DistanceMatrix stand-in computed by the oracle BFS (for host-only tests)."""

    def __init__(self, g):
        self.graph = g
        self._d = ot.server_hops(g.n_nodes, g.links.tolist(), g.n_servers)

    def server_numpy(self):
        return self._d


class HostCost:
    def __init__(self, p):
        self.p_np = np.asarray(p)

    def numpy(self):
        return self.p_np

    @property
    def S(self):
        return self.p_np.shape[1]


# ---------------- topology ----------------

def test_spec_sizes_and_kinds():
    for kind in topo.KINDS:
        g = topo.build_topology(topo.TopologySpec(kind, 16, 4, 4))
        assert g.n_devices == 256 and g.n_servers == 64
        assert (np.bincount(g.device_server) == 4).all()
        # every server has exactly one link, to its leaf
        for s in range(g.n_servers):
            nb = [b if a == s else a for a, b in g.links.tolist() if s in (a, b)]
            assert nb == [int(g.server_leaf[s])]


def test_topology_spec_validation():
    with pytest.raises(ConfigError):
        topo.TopologySpec("Torus", 2, 2, 2)
    with pytest.raises(ConfigError):
        topo.TopologySpec("FatTree", 0, 2, 2)
    with pytest.raises(ConfigError):
        topo.build_topology(topo.TopologySpec("DragonflySparse", 2, 1, 1))


def test_fattree_block_structure():
    """Acceptance #5: 256-device FatTree: intra-server 0, intra-leaf equal, cross-leaf equal and larger."""
    g = topo.build_topology(topo.TopologySpec("FatTree", 16, 4, 4))
    d = ot.device_hops(ot.server_hops(g.n_nodes, g.links.tolist(), g.n_servers), g.device_server)
    leaf = g.server_leaf[g.device_server]
    same_srv = g.device_server[:, None] == g.device_server[None, :]
    same_leaf = (leaf[:, None] == leaf[None, :]) & ~same_srv
    cross = leaf[:, None] != leaf[None, :]
    assert (d[same_srv] == 0).all()
    assert len(set(d[same_leaf].tolist())) == 1 and len(set(d[cross].tolist())) == 1
    assert d[cross].max() > d[same_leaf].max()
    gd = topo.build_topology(topo.TopologySpec("Dragonfly", 16, 4, 4))
    dd = ot.device_hops(ot.server_hops(gd.n_nodes, gd.links.tolist(), gd.n_servers), gd.device_server)
    assert len(set(dd[dd > 0].tolist())) >= 3
    # Dragonfly has strictly more distinct off-diagonal values than FatTree
    assert len(set(dd[dd > 0].tolist())) > len(set(d[d > 0].tolist()))


def test_sparse_dragonfly_diameter():
    """ring + diameter chord has leaf diameter < 8 (the plain 16-ring)."""
    g = topo.build_topology(topo.TopologySpec("DragonflySparse", 16, 1, 1))
    d = ot.server_hops(g.n_nodes, g.links.tolist(), g.n_servers)
    assert d.max() - 2 < 8


def test_distance_invariants_all_kinds():
    for kind in topo.KINDS + topo.EXTENSION_KINDS:
        leaves = 18 if kind == "SlimFly" else 16
        g = topo.build_topology(topo.TopologySpec(kind, leaves, 2, 2))
        d = ot.device_hops(ot.server_hops(g.n_nodes, g.links.tolist(), g.n_servers), g.device_server)
        assert (d == d.T).all() and (np.diag(d) == 0).all()
        off = ~(g.device_server[:, None] == g.device_server[None, :])
        assert (d[off] >= 2).all()
        # triangle inequality
        assert (d[:, None, :] <= d[:, :, None] + d[None, :, :]).all()


def test_slimfly_diameter_two():
    for n in (18, 50):
        g = topo.build_topology(topo.TopologySpec("SlimFly", n, 1, 1))
        d = ot.server_hops(g.n_nodes, g.links.tolist(), g.n_servers)
        assert d.max() - 2 <= 2  # router graph diameter 2


def test_topology_json_roundtrip(tmp_path):
    g = topo.build_topology(topo.TopologySpec("FatTreeHier", 8, 2, 2))
    topo.save_topology(g, tmp_path / "t.json")
    h = topo.load_topology(tmp_path / "t.json")
    assert np.array_equal(g.links, h.links) and np.array_equal(g.device_server, h.device_server)
    assert g.switch_kind == h.switch_kind


def test_locality_order():
    # 1 leaf, 2 servers x 2 GPUs -> [s0g0, s0g1, s1g0, s1g1]
    g = topo.build_topology(topo.TopologySpec("FatTree", 1, 2, 2))
    assert topo.locality_order(g, HostDist(g)) == [0, 1, 2, 3]
    # ring: consecutive leaves ring-adjacent except at the single seam
    g = topo.build_topology(topo.TopologySpec("DragonflySparse", 16, 1, 1))
    o = topo.locality_order(g, HostDist(g))
    assert sorted(o) == list(range(16))
    leaves = [g.server_leaf[g.device_server[d]] - g.n_servers for d in o]
    adj = {(int(a), int(b)) for a, b in g.links.tolist()}
    nonadj = sum((min(a, b) + g.n_servers, max(a, b) + g.n_servers) not in adj for a, b in zip(leaves, leaves[1:]))
    assert nonadj <= 1


def test_default_attention_placement(tmp_path):
    m = mt.ModelSpec(4, 8, 2)
    a = mt.default_attention_placement(m, [3, 1, 2, 0])
    assert a.dispatch.tolist() == [3, 1, 2, 0] and a.collect.tolist() == [1, 2, 0, 0]
    a = mt.default_attention_placement(mt.ModelSpec(2, 4, 1), [5])
    assert a.dispatch.tolist() == [5, 5] and a.collect.tolist() == [5, 5]


# ---------------- placers / validate ----------------

def test_rr_window_and_wrap():
    m = mt.ModelSpec(1, 4, 1)
    order = list(range(8))
    attn = mt.AttentionPlacement([0], [0])
    p = mpl.place_round_robin(m, attn, order, mpl.Constraints(4, 1))
    assert sorted(p.assign[0].tolist()) == [0, 1, 6, 7]
    assert p.assign[0].tolist() == [6, 7, 0, 1]
    # E = c_layer -> all on the dispatch device
    p = mpl.place_round_robin(mt.ModelSpec(1, 4, 1), mt.AttentionPlacement([3], [3]), order, mpl.Constraints(4, 4))
    assert p.assign[0].tolist() == [3, 3, 3, 3]
    # E=4, c_layer=2, d=2: window [i-1, i+1) (the stated convention)
    p = mpl.place_round_robin(m, mt.AttentionPlacement([4], [4]), order, mpl.Constraints(4, 2))
    assert p.assign[0].tolist() == [3, 3, 4, 4]


def test_rr_c_exp_infeasible():
    m = mt.ModelSpec(3, 4, 1)
    with pytest.raises(InfeasibleError):
        mpl.place_round_robin(m, mt.AttentionPlacement([0, 0, 0], [0, 0, 0]), list(range(4)), mpl.Constraints(2, 1))


def test_greedy_examples():
    m = mt.ModelSpec(1, 2, 1)
    p = mpl.place_greedy(m, None, HostCost([[0, 4]]), mpl.Constraints(2, 1))
    assert p.assign.tolist() == [[0, 1]]
    m = mt.ModelSpec(2, 3, 1)
    p = mpl.place_greedy(m, None, HostCost([[5, 5, 5], [5, 5, 5]]), mpl.Constraints(10, 10))
    assert (p.assign == 0).all()
    with pytest.raises(InfeasibleError):
        mpl.place_greedy(mt.ModelSpec(2, 2, 1), None, HostCost([[0, 1], [0, 1]]), mpl.Constraints(1, 1))


def test_greedy_pointwise_minimal_replay():
    rng = np.random.default_rng(4)
    L, E, S = 5, 12, 8
    p = rng.integers(0, 10, (L, S))
    c = mpl.Constraints(9, 2)
    pl = mpl.place_greedy(mt.ModelSpec(L, E, 1), None, HostCost(p), c)
    used = np.zeros(S, int)
    for l in range(L):
        lu = np.zeros(S, int)
        for e in range(E):
            ok = [s for s in range(S) if lu[s] < c.c_layer and used[s] < c.c_exp]
            best = min(ok, key=lambda s: (p[l, s], s))
            assert pl.assign[l, e] == best
            lu[best] += 1
            used[best] += 1


def test_validate_families():
    m = mt.ModelSpec(1, 3, 1)
    c = mpl.Constraints(3, 1)
    v = mpl.validate(mpl.Placement(np.array([[0, 0, 0]])), c, m, 3)
    assert any(x.family == "c_layer" and x.device == 0 and x.count == 3 for x in v)
    assert mpl.validate(mpl.Placement(np.array([[0, 1, 2]])), c, m, 3) == []
    v = mpl.validate(mpl.Placement(np.array([[0, 1, 7]])), c, m, 3)
    assert any(x.family == "assignment" and x.expert == 2 for x in v)
    v = mpl.validate(mpl.Placement(np.array([[0, 1, 2], [0, 1, 2]])), mpl.Constraints(1, 1), mt.ModelSpec(2, 3, 1), 3)
    assert {x.family for x in v} == {"c_exp"}


def test_placement_csv_roundtrip(tmp_path):
    a = np.arange(12).reshape(3, 4) % 5
    mpl.write_placement(mpl.Placement(a), tmp_path / "p.csv")
    assert (tmp_path / "p.csv").read_text().splitlines()[0] == "layer,expert,device"
    b = mpl.read_placement(tmp_path / "p.csv", mt.ModelSpec(3, 4, 1), mpl.Constraints(12, 4), 5)
    assert np.array_equal(a, b.assign)
    with pytest.raises(MoeplaceError):
        mpl.read_placement(tmp_path / "p.csv", mt.ModelSpec(3, 4, 1), mpl.Constraints(2, 1), 5)


def test_constraints_feasibility():
    with pytest.raises(ConfigError):
        mpl.Constraints(1, 2)
    c = mpl.Constraints(54, 1)
    with pytest.raises(InfeasibleError):
        c.check_feasible(mt.ModelSpec(27, 64, 6), 32)  # S*c_layer < E
    mpl.Constraints(54, 2).check_feasible(mt.ModelSpec(27, 64, 6), 32)


# ---------------- solver (native host min-cost flow) ----------------

def _inst(w, c_layer, c_exp, p=None):
    w = np.asarray(w, dtype=np.float64)
    L, E, S = w.shape
    return sv.PlacementInstance(w, None, mpl.Constraints(c_exp, c_layer), L, E, S, p, scale=1.0)


def test_solver_spec_examples():
    pl, obj = sv.solve_exact(_inst([[[3, 1]]], 1, 1))
    assert pl.assign.tolist() == [[1]] and obj == 1
    pl, obj = sv.solve_exact(_inst([[[0, 5], [0, 5]]], 1, 1))
    assert obj == 5
    with pytest.raises(InfeasibleError):
        sv.solve_exact(_inst([[[0, 5], [0, 5], [1, 1]]], 1, 1))


def test_solver_equals_brute_force_100_instances():
    """Acceptance #1: >= 100 seeded random tiny instances, solve_exact == brute_force_optimum."""
    rng = np.random.default_rng(2024)
    done = 0
    while done < 100:
        L, E, S = int(rng.integers(1, 4)), int(rng.integers(1, 5)), int(rng.integers(1, 6))
        if S ** (L * E) > 10 ** 5:
            continue
        c_layer = int(rng.integers(1, E + 1))
        c_exp = int(rng.integers(c_layer, L * E + 1))
        if S * c_layer < E or S * c_exp < L * E:
            continue
        inst = _inst(rng.integers(0, 20, (L, E, S)), c_layer, c_exp)
        try:
            bf = sv.brute_force_optimum(inst)
        except InfeasibleError:
            with pytest.raises(InfeasibleError):
                sv.solve_exact(inst)
            done += 1
            continue
        pl, obj = sv.solve_exact(inst)
        assert obj == bf
        assert mpl.validate(pl, inst.constraints, mt.ModelSpec(L, E, 1), S) == []
        done += 1


def test_solver_compressed_network_matches_highs():
    """Class-compressed network (w = f*p) vs scipy HiGHS LP on the full network, with c_exp binding
    (one network over all layers) and slack (L*c_layer <= c_exp: independent per-layer flows)."""
    from scipy.optimize import linprog
    from scipy.sparse import lil_matrix
    rng = np.random.default_rng(7)
    for trial in range(4):
        L, E, S = 3, 6, 5
        p = rng.integers(0, 5, (L, S)).astype(np.uint8)
        f = rng.random((L, E))
        f /= f.sum(axis=1, keepdims=True)
        w, wi = ot.coefficients(f, p)
        c = mpl.Constraints(5, 2) if trial % 2 == 0 else mpl.Constraints(6, 2)
        inst = sv.PlacementInstance(w, wi, c, L, E, S, p)
        pl, obj = sv.solve_exact(inst)
        n = L * E * S
        A_eq = lil_matrix((L * E, n))
        for i in range(L * E):
            A_eq[i, i * S:(i + 1) * S] = 1
        rows = []
        for l in range(L):
            for s in range(S):
                r = np.zeros(n)
                r[[((l * E + e) * S + s) for e in range(E)]] = 1
                rows.append((r, c.c_layer))
        for s in range(S):
            r = np.zeros(n)
            r[[((l * E + e) * S + s) for l in range(L) for e in range(E)]] = 1
            rows.append((r, c.c_exp))
        res = linprog(wi.ravel().astype(float), A_ub=np.array([r for r, _ in rows]), b_ub=[b for _, b in rows],
                      A_eq=A_eq.tocsr(), b_eq=np.ones(L * E), bounds=(0, 1), method="highs")
        assert res.status == 0
        assert pl.solve_report["objective_scaled"] == round(res.fun)
        # the compressed network gives the same optimum as the uncompressed one
        inst2 = sv.PlacementInstance(w, wi, c, L, E, S, None)
        _, obj2 = sv.solve_exact(inst2)
        assert abs(obj2 - obj) <= 1e-12 * max(1.0, obj)


def test_solver_monotone_in_c_layer():
    """Acceptance #7: optimum non-increasing as c_layer relaxes (c_layer in {1, 4, 8})."""
    rng = np.random.default_rng(1)
    L, E, S = 4, 16, 16
    p = rng.integers(0, 9, (L, S)).astype(np.uint8)
    f = rng.random((L, E))
    f /= f.sum(axis=1, keepdims=True)
    w, wi = ot.coefficients(f, p)
    objs = [sv.solve_exact(sv.PlacementInstance(w, wi, mpl.Constraints(16, cl), L, E, S, p))[1] for cl in (1, 4, 8)]
    assert objs[0] >= objs[1] >= objs[2]


def test_flow_network_shape():
    inst = _inst(np.ones((2, 3, 4)), 2, 3)
    net = sv.flow_network(inst)
    assert net.n_nodes == 1 + 6 + 8 + 4 + 1
    assert len(net.arcs) == 6 + 6 * 4 + 8 + 4


def test_brute_force_guard():
    with pytest.raises(ConfigError):
        sv.brute_force_optimum(_inst(np.ones((3, 4, 5)), 1, 4))


# ---------------- trace text format: the oracle's restatement (the product parses on the device) ----

def _write(path, lines):
    path.write_text("\n".join(lines) + "\n")


def test_oracle_text_parser_errors(tmp_path):
    from oracle.textio import TextParseError, parse_text
    f = tmp_path / "t.txt"
    _write(f, ["#moeplace-trace v1 L=2 E=4 K=2", "0\tlayer0:0,1\tlayer1:2,3", "0\tlayer0:0,4\tlayer1:2,3"])
    with pytest.raises(TextParseError) as e:
        parse_text(f)  # expert index E -> error at that line
    assert e.value.line_no == 3
    _write(f, ["#moeplace-trace v1 L=2 E=4 K=2", "0\tlayer0:0,1"])
    with pytest.raises(TextParseError) as e:
        parse_text(f)
    assert e.value.line_no == 2
    _write(f, ["#moeplace-trace v1 L=2 E=4 K=2", "0\tlayer0:0,1\tlayer1:2,2"])
    with pytest.raises(TextParseError):
        parse_text(f)
    _write(f, ["garbage"])
    with pytest.raises(TextParseError) as e:
        parse_text(f)
    assert e.value.line_no == 1
    f.write_text("")
    assert parse_text(f)[1].shape[0] == 0


def test_oracle_text_roundtrip(tmp_path):
    from oracle.textio import parse_text, regroup, write_text
    f = tmp_path / "t.txt"
    lines = ["#moeplace-trace v1 L=2 E=5 K=2", "0\tlayer0:0,1\tlayer1:2,3", "0\tlayer0:4,1\tlayer1:0,3",
             "3\tlayer0:2,1\tlayer1:2,4"]
    _write(f, lines)
    shape, sel, cid = parse_text(f)
    sel2, ids, bounds = regroup(sel, cid)
    assert sel.shape[0] == 3 and ids.tolist() == [0, 3] and bounds.tolist() == [0, 2, 3]
    g = tmp_path / "u.txt"
    write_text(g, shape, sel2, np.repeat(ids, np.diff(bounds)))
    assert g.read_text() == f.read_text()
    _write(f, ["#moeplace-trace v1 L=1 E=3 K=1", "1\t0:2"])  # prefix-less fields are accepted
    assert parse_text(f)[1].tolist() == [[[2]]]


def test_product_has_no_host_text_engine(tmp_path):
    """The product parses and writes traces on the device only (no CPU fallback): asking for a
    host engine is a configuration error, not a silent CPU path."""
    f = tmp_path / "t.txt"
    _write(f, ["#moeplace-trace v1 L=1 E=3 K=1", "1\t0:2"])
    with pytest.raises(ConfigError):
        mt.parse_trace(f, engine="host")
    tr = mt.ActivationTrace(mt.ModelSpec(1, 3, 1), None, 0, 0, np.zeros(0, np.int64), np.zeros(1, np.int64))
    with pytest.raises(ConfigError):
        mt.write_trace(tr, tmp_path / "u.txt", engine="host")


def test_cli_config_and_placement_errors_map_to_exit_codes(tmp_path):
    """an invalid or non-object --config exits 2 (config error), a malformed placement
    CSV row raises TraceParseError with its line number (exit 4)."""
    import moeplace.cli as cli
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert cli.main(["topo", "build", "--config", str(bad), "--out", str(tmp_path / "g.json")]) == 2
    bad.write_text("[1, 2]")
    assert cli.main(["topo", "build", "--config", str(bad), "--out", str(tmp_path / "g.json")]) == 2
    ok = tmp_path / "ok.json"
    ok.write_text('{"L": 2, "E": 4, "K": 2, "c_exp": 4, "topology": "FatTree", "num_leaf_switches": 2, '
                  '"num_nodes_per_leaf": 1, "num_gpus_per_server": 2}')
    assert cli.main(["topo", "build", "--config", str(ok), "--out", str(tmp_path / "g.json")]) == 0
    csvf = tmp_path / "p.csv"
    csvf.write_text("layer,expert,device\n0,0,1\n0,1\n")
    with pytest.raises(TraceParseError) as e:
        mpl.read_placement(csvf, mt.ModelSpec(1, 2, 1))
    assert e.value.line_no == 3 and exit_code(e.value) == 4
    csvf.write_text("layer,expert,device\n0,x,1\n")
    with pytest.raises(TraceParseError) as e:
        mpl.read_placement(csvf, mt.ModelSpec(1, 2, 1))
    assert e.value.line_no == 2


def test_split_trace_host():
    tr = mt.ActivationTrace(mt.ModelSpec(1, 2, 1), None, 0, 10, np.arange(4), np.array([0, 2, 5, 7, 10]))
    a, b = mt.split_trace(tr, 2, 1)
    assert (a.tok_begin, a.n_tokens, b.tok_begin, b.n_tokens) == (0, 5, 5, 2)
    assert a.chunk_ids.tolist() == [0, 1] and b.chunk_ids.tolist() == [2]
    with pytest.raises(ConfigError):
        mt.split_trace(tr, 3, 2)


def test_chunk_bounds_even():
    b = mt.chunk_bounds_even(10, 3)
    lab = np.repeat(np.arange(3), np.diff(b))
    assert np.array_equal(lab, np.arange(10) * 3 // 10)
    assert mt.chunk_bounds_even(2, 5).tolist() == [0, 1, 1, 2, 2, 2]


def test_generator_host_params_match_oracle():
    from oracle import gen as og
    for seed in (0, 1, 2 ** 40 + 3):
        assert np.array_equal(mt.layer_permutations(seed, 3, 256).astype(np.int64), og.perms(seed, 3, 256))
    for s in (0.0, 1.2, 2.0):
        assert np.array_equal(mt.zipf_cdf(64, s).astype(np.int64), og.cdf(64, s))
        assert int(mt.zipf_cdf(256, s)[-1]) < 2 ** 31


def test_model_spec_validation():
    with pytest.raises(ConfigError):
        mt.ModelSpec(1, 4, 5)
    with pytest.raises(ConfigError):
        mt.ModelSpec(0, 4, 1)


# ---------------- cli / config / errors ----------------

def test_config_rejects_unknown_keys(tmp_path):
    with pytest.raises(ConfigError):
        cli.ExperimentConfig.from_dict({"L": 2, "E": 4, "K": 1, "c_exp": 8, "bogus": 1})
    with pytest.raises(ConfigError):
        cli.ExperimentConfig.from_dict({"L": 2, "E": 4, "K": 1})
    with pytest.raises(ConfigError):
        cli.ExperimentConfig.from_dict({"L": 2, "E": 4, "K": 1, "c_exp": 8, "methods": ["magic"]})
    f = tmp_path / "c.json"
    f.write_text(json.dumps({"L": 2, "E": 4, "K": 1, "c_exp": 8, "oops": 3}))
    assert cli.main(["compare", "--config", str(f)]) == 2


def test_exit_codes():
    assert exit_code(ConfigError("x")) == 2
    assert exit_code(InfeasibleError("x")) == 3
    assert exit_code(TraceParseError("x", 3)) == 4
    assert exit_code(TopologyError("x")) == 2
    assert str(TraceParseError("bad", 7)) == "line 7: bad" and TraceParseError("bad", 7).line_no == 7
    assert issubclass(TopologyError, MoeplaceError)


def test_perturb_swaps_keep_constraints():
    rng = np.random.default_rng(0)
    L, E, S = 6, 16, 16
    base = np.stack([rng.permutation(S) for _ in range(L)]).astype(np.int32)
    c = mpl.Constraints(6, 1)
    cand = mpl.perturb_swaps(mpl.Placement(base), 20, 8, seed0=1000)
    assert cand.shape == (20, L, E)
    for i in range(20):
        assert mpl.validate(mpl.Placement(cand[i]), c, mt.ModelSpec(L, E, 1), S) == []
        assert (np.sort(cand[i], axis=1) == np.sort(base, axis=1)).all()
    again = mpl.perturb_swaps(mpl.Placement(base), 20, 8, seed0=1000)
    assert np.array_equal(cand, again)


def test_dedup_oracle_hand_example():
    from oracle import evaluate as oe
    # one token, L=1, K=4 picks on devices of servers [0, 1, 1, 2]; dispatch server 0
    sel = np.array([[[0, 1, 2, 3]]], dtype=np.uint8)
    pe = np.array([[0, 4, 4, 6]])
    srv_e = np.array([[0, 1, 1, 2]])
    h, u, d = oe.dedup_sums(sel, pe, srv_e, np.array([0]), np.array([0, 1]))
    assert h.tolist() == [14] and u.tolist() == [2] and d.tolist() == [10]


def test_cpu_fused_pass_matches_separate():
    from oracle import evaluate as oe
    from oracle import gen as og
    from oracle import stats as ost
    sel, b = og.generate(5, 32, 4, 1.2, 3000, 7, 2)
    rng = np.random.default_rng(1)
    pes = [oe.pe_table(rng.integers(0, 200, (5, 8)), rng.integers(0, 8, (5, 32))) for _ in range(6)]
    cnt, sums = oe.fused_pass(sel, pes, b, 32)
    assert np.array_equal(cnt, ost.counts(sel, 32))
    for q in range(6):
        assert np.array_equal(sums[q], oe.chunk_sums(sel, pes[q], b))


def test_batched_reports_equal_single_reports():
    """reports_from_sums (evaluate_many's batched float derivation) gives the same EvalReports, bit
    for bit, as report_from_sums per placement, with empty chunks and large sums."""
    import moeplace.eval as ev
    rng = np.random.default_rng(7)
    for P, C in [(1, 1), (3, 17), (64, 150), (9, 401)]:
        sums = rng.integers(0, 10 ** 12, (P, C))
        tok = rng.integers(0, 7000, C)
        if C > 1:
            tok[rng.integers(1, C)] = 0
        tok[0] = max(tok[0], 1)
        sums[:, tok == 0] = 0
        labels = [f"p{i}" for i in range(P)]
        batched = ev.reports_from_sums(sums, tok, labels)
        assert batched == [ev.report_from_sums(sums[i], tok, labels[i]) for i in range(P)]
