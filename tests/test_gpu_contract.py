"""The tensor-core contraction (tcgen05 kind::i8, mp_contract_tc_u8) and the device search-loop
kernels (pe gather, swap perturbation, batch objectives, accept), bit-exact against independent
references: numpy, the CUDA-core int64 contraction mp_contract_counts, and float64 GEMMs whose
integer partial sums stay below 2^53 (exact)."""
import numpy as np
import pytest

import moeplace.eval as ev
import moeplace.model_trace as mt
import moeplace.placement as mpl
from moeplace.errors import MoeplaceError
from paper_2508_09229_b200 import _lib

from helpers import random_assign, setup_topology

pytestmark = pytest.mark.gpu


def _exact_ref(pe, cnt):
    """int64 pe @ cnt^T via float64 on the device: every partial sum is an integer < 2^53 here."""
    import torch
    r = pe.to(torch.float64) @ cnt.to(torch.float64).T
    assert float(r.abs().max()) < 2 ** 53
    return r.to(torch.int64)


@pytest.mark.parametrize("P,LE,C,cmax", [
    (1, 64, 1, 255), (100, 1000, 7, 255), (128, 1024, 150, 6667), (129, 1728, 33, 70000),
    (4096, 14848, 150, 6667),            # BASELINE config 4 shape (R1 L*E, 150 chunks, 2 digits)
    (300, 14848, 300, 6667),             # C*ndig = 600 > 512: two N tiles
    (64, 40000, 5, 255),                 # L*E > 32768: split-K forced for int32 exactness
    (40, 4096, 9, 2 ** 30),              # 4 digits
])
def test_contract_tc_matches_exact_references(P, LE, C, cmax):
    import torch
    rng = np.random.default_rng(P * 7 + C)
    pe = torch.as_tensor(rng.integers(0, 256, (P, LE)).astype(np.uint8), device="cuda")
    cnt = torch.as_tensor(rng.integers(0, cmax + 1, (C, LE)), device="cuda")
    cnt[0, 0] = cmax
    want = _exact_ref(pe, cnt)
    got = ev.contract_tc(cnt, pe, max_count=cmax)
    assert torch.equal(got, want)
    d = ev.CountDigits(cnt, cmax)
    # single CTAs: stream-K splits landing anywhere inside the pe tiles; negative: CTA pairs
    # (tcgen05 cta_group::2, 256-row tiles), including pairs that straddle tiles
    for ctas in (1, 3, 77, 300, -1, -3, -37):
        out = torch.zeros((P, C), dtype=torch.int64, device="cuda")
        d.contract(pe, out, ctas=ctas)
        assert torch.equal(out, want), ctas
    d.check()
    if P * LE * C <= 4096 * 14848 * 150:
        cc = torch.zeros((P, C), dtype=torch.int64, device="cuda")
        pe_c = pe.contiguous()
        _lib.call("mp_contract_counts", _lib.ptr(cnt), C, _lib.ptr(pe_c), P, LE, _lib.ptr(cc), _lib.stream_handle())
        assert torch.equal(cc, want)


def test_contract_tc_accumulates_and_takes_padded_views():
    import torch
    rng = np.random.default_rng(5)
    P, LE, C = 50, 1000, 6
    buf = torch.zeros((P, 1008), dtype=torch.uint8, device="cuda")
    buf[:, :LE] = torch.as_tensor(rng.integers(0, 256, (P, LE)).astype(np.uint8), device="cuda")
    pe = buf[:, :LE]  # 16-byte pitch view: used in place, no copy
    cnt = torch.as_tensor(rng.integers(0, 300, (C, LE)), device="cuda")
    d = ev.CountDigits(cnt, 299)
    out = torch.full((P, C), 7, dtype=torch.int64, device="cuda")
    d.contract(pe, out)
    assert torch.equal(out, _exact_ref(pe, cnt) + 7)  # accumulate-into, like every other kernel


def test_pe_gather_multi_topology_and_errors():
    import torch
    m = mt.ModelSpec(6, 40, 4)
    tops = [setup_topology("FatTree", 4, 2, 4, m), setup_topology("Dragonfly", 4, 2, 2, m),
            setup_topology("DragonflySparse", 4, 2, 4, m)]
    rng = np.random.default_rng(2)
    pls, costs = [], []
    for i in range(9):
        tt = tops[i % 3]
        pls.append(mpl.Placement(random_assign(rng, m.L, m.E, tt[0].n_devices)))
        costs.append(tt[4])
    pe = ev.pe_matrix(pls, costs, m).cpu().numpy()
    for q, (pl, c) in enumerate(zip(pls, costs)):
        p = c.numpy()
        assert np.array_equal(pe[q].reshape(m.L, m.E), p[np.arange(m.L)[:, None], pl.assign]), q
    bad = pls[4].assign.copy()
    bad[2, 3] = costs[4].S  # one past the end of ITS topology (narrower than the widest)
    with pytest.raises(MoeplaceError, match="placement 4"):
        ev.pe_matrix(pls[:4] + [mpl.Placement(bad)] + pls[5:], costs, m)
    with pytest.raises(MoeplaceError):
        ev.evaluate_batch(mt.generate_trace(m, 1.2, 500, 3, 1), np.stack([p.assign for p in pls[:4]] + [bad]),
                          costs[:5])


def test_perturbation_objective_and_accept_kernels():
    """mp_perturb_pe_u8 rows == the incumbent row with the recorded swaps replayed in numpy;
    mp_batch_objective == the EvalReport floats (mean exactly; std / max to 1e-12); mp_search_accept
    picks the lowest-index argmin and replays its swaps on the assignment and the cost row."""
    import torch
    m = mt.ModelSpec(58, 256, 8)
    g, dist, order, attn, cost = setup_topology("Dragonfly", 16, 4, 4, m)
    rr = mpl.place_round_robin(m, attn, order, mpl.Constraints(64, 1))
    LE, ldpe, B, ns = m.L * m.E, m.L * m.E, 64, 5
    pe_cur = ev.pe_matrix([rr], cost, m)[0].contiguous()
    pe_b = torch.empty((B, ldpe), dtype=torch.uint8, device="cuda")
    sw = torch.empty((B, ns, 3), dtype=torch.int32, device="cuda")
    sh = _lib.stream_handle()
    _lib.call("mp_perturb_pe_u8", _lib.ptr(pe_cur), m.L, m.E, B, ns, 1234, 7, _lib.ptr(pe_b), ldpe, _lib.ptr(sw), sh)
    rows, swaps, base = pe_b.cpu().numpy(), sw.cpu().numpy(), pe_cur.cpu().numpy()
    for b in range(B):
        r = base.copy().reshape(m.L, m.E)
        for l, x, y in swaps[b]:
            r[l, x], r[l, y] = r[l, y], r[l, x]
        assert np.array_equal(rows[b], r.ravel()), b
    assert len({tuple(s.ravel()) for s in swaps}) == B  # distinct draws per candidate
    # objectives
    tr = mt.generate_trace(m, 1.2, 30_000, 40, 2)
    tok = tr.chunk_token_counts().copy()
    sums = torch.as_tensor(np.random.default_rng(1).integers(0, 10 ** 7, (B, 40)), device="cuda")
    sums[:, 5] = 0
    tok_d = torch.as_tensor(tok, device="cuda")
    rep_tok = tok.copy()
    for kind in (0, 1, 2):
        obj = torch.empty(B, dtype=torch.float64, device="cuda")
        _lib.call("mp_batch_objective", _lib.ptr(sums), _lib.ptr(tok_d), B, 40, kind, 0.5, _lib.ptr(obj), sh)
        reps = ev.reports_from_sums(sums.cpu().numpy(), rep_tok, [""] * B)
        means = sums.cpu().numpy() / tok
        o = obj.cpu().numpy()
        for b, r in enumerate(reps):
            want = {0: r.mean_hops_per_token, 1: r.mean_hops_per_token + 0.5 * r.std_hops, 2: means[b].max()}[kind]
            assert (o[b] == want) if kind == 0 else abs(o[b] - want) <= 1e-12 * want
    # accept: the lowest-index minimum wins and its swaps are replayed
    obj = torch.full((B,), 10.0, dtype=torch.float64, device="cuda")
    obj[17], obj[40] = 3.0, 3.0
    assign = torch.as_tensor(rr.assign, device="cuda").to(torch.int32).contiguous()
    cur = torch.tensor([5.0], dtype=torch.float64, device="cuda")
    hist = torch.zeros(4, dtype=torch.float64, device="cuda")
    acc = torch.zeros(4, dtype=torch.int64, device="cuda")
    pe_in = pe_cur.clone()
    _lib.call("mp_search_accept", _lib.ptr(obj), B, _lib.ptr(sw), ns, m.E, _lib.ptr(assign), _lib.ptr(pe_in),
              _lib.ptr(cur), _lib.ptr(hist), 1, _lib.ptr(acc), sh)
    assert acc[1].item() == 17 and cur.item() == 3.0 and hist[1].item() == 3.0
    assert np.array_equal(pe_in.cpu().numpy(), rows[17])
    a = rr.assign.copy()
    for l, x, y in swaps[17]:
        a[l, x], a[l, y] = a[l, y], a[l, x]
    assert np.array_equal(assign.cpu().numpy(), a)
    _lib.call("mp_search_accept", _lib.ptr(obj), B, _lib.ptr(sw), ns, m.E, _lib.ptr(assign), _lib.ptr(pe_in),
              _lib.ptr(cur), _lib.ptr(hist), 2, _lib.ptr(acc), sh)
    assert acc[2].item() == -1 and hist[2].item() == 3.0  # no strict improvement: incumbent kept


def test_objective_value_on_device_matches_numpy():
    m = mt.ModelSpec(27, 64, 6)
    g, dist, order, attn, cost = setup_topology("FatTree", 2, 2, 8, m)
    tr = mt.generate_trace(m, 1.2, 20_000, 10, 4)
    f = mt.estimate_frequencies(tr, m)
    rng = np.random.default_rng(0)
    pl = mpl.Placement(random_assign(rng, m.L, m.E, g.n_devices))
    p = cost.numpy()
    pe = p[np.arange(m.L)[:, None], pl.assign].astype(np.float64)
    want = float(np.sum(f.f * pe))
    got = ev.objective_value(pl, f, cost)                       # exact integer contraction / (K N)
    assert abs(got - want) <= 1e-12 * want
    assert got == int((f.counts * pe.astype(np.int64)).sum()) / (6 * 20_000)
    ff = mt.FrequencyTable(f.f.copy())                          # float-only frequencies
    assert abs(ev.objective_value(pl, ff, cost) - want) <= 1e-12 * want
