"""Oracle traffic evaluator (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

SPEC.md:336-379:
  token_hops(t)   = sum_l sum_{e in topK(t,l)} p[l, assign[l, e]]
  evaluate        = per-chunk integer hop sums; mean = sum / n_tokens; std = population std of the
                    per-chunk means, empty chunks excluded and counted
  objective_value = sum_{l,e} f[l,e] * p[l, assign[l,e]]
  gain            = 100 * (baseline - method) / method
  communication_map: per activation, D(d_l, s) -> (srv d_l, srv s) and D(s, c_l) -> (srv s, srv c_l),
                    symmetrised as (M + M^T)/2, divided by the token count
"""
from __future__ import annotations

import numba as nb
import numpy as np


def pe_table(p: np.ndarray, assign: np.ndarray) -> np.ndarray:
    """pe[l, e] = p[l, assign[l, e]] (int64)."""
    L = assign.shape[0]
    return p.astype(np.int64)[np.arange(L)[:, None], assign]


@nb.njit(cache=True)
def token_hops(sel_t, pe):
    """sel_t: [L, K] selections of one token."""
    L, K = sel_t.shape
    s = 0
    for l in range(L):
        for k in range(K):
            s += pe[l, sel_t[l, k]]
    return s


@nb.njit(cache=True, parallel=True)
def _chunk_sums(sel, pe, bounds, t0):
    C = bounds.shape[0] - 1
    L = sel.shape[1]
    K = sel.shape[2]
    out = np.zeros(C, dtype=np.int64)
    for c in nb.prange(C):
        lo = max(bounds[c], t0) - t0
        hi = min(bounds[c + 1], t0 + sel.shape[0]) - t0
        s = 0
        for t in range(lo, hi):
            for l in range(L):
                for k in range(K):
                    s += pe[l, sel[t, l, k]]
        out[c] = s
    return out


def chunk_sums(sel: np.ndarray, pe: np.ndarray, bounds: np.ndarray, t0: int = 0) -> np.ndarray:
    """Exact int64 hop sums per chunk; ``sel`` holds tokens [t0, t0 + N) of the bounds' numbering."""
    return _chunk_sums(np.ascontiguousarray(sel), np.ascontiguousarray(pe, dtype=np.int64),
                       np.asarray(bounds, dtype=np.int64), np.int64(t0))


@nb.njit(cache=True, parallel=True)
def _token_sums(sel, pe):
    N, L, K = sel.shape
    out = np.zeros(N, dtype=np.int64)
    for t in nb.prange(N):
        s = 0
        for l in range(L):
            for k in range(K):
                s += pe[l, sel[t, l, k]]
        out[t] = s
    return out


def per_token_hops(sel: np.ndarray, pe: np.ndarray) -> np.ndarray:
    return _token_sums(np.ascontiguousarray(sel), np.ascontiguousarray(pe, dtype=np.int64))


def report(sums: np.ndarray, tokens: np.ndarray) -> dict:
    """EvalReport floats from integer per-chunk sums and token counts."""
    sums = np.asarray(sums, dtype=np.int64)
    tokens = np.asarray(tokens, dtype=np.int64)
    keep = tokens > 0
    n = int(tokens.sum())
    total = int(sums.sum())
    means = sums[keep] / tokens[keep]
    return {"mean": total / n, "std": float(np.std(means)), "n_tokens": n, "n_chunks": int(keep.sum()),
            "empty_chunks": int((~keep).sum()), "hop_sum": total}


def objective(f: np.ndarray, pe: np.ndarray) -> float:
    return float(np.sum(f * pe.astype(np.float64)))


def gain(baseline: float, method: float) -> float:
    if not method > 0:
        raise ValueError("method_hops must be positive")
    return 100.0 * (baseline - method) / method


def comm_map(cnt: np.ndarray, assign: np.ndarray, device_server: np.ndarray, dsrv: np.ndarray,
             dispatch: np.ndarray, collect: np.ndarray, n_tokens: int):
    """(symmetrised float map, raw int64 directed map) from per-(l, e) counts."""
    n = dsrv.shape[0]
    raw = np.zeros((n, n), dtype=np.int64)
    L, E = cnt.shape
    for l in range(L):
        a = int(device_server[dispatch[l]])
        b = int(device_server[collect[l]])
        for e in range(E):
            c = int(cnt[l, e])
            if c == 0:
                continue
            s = int(device_server[assign[l, e]])
            raw[a, s] += c * int(dsrv[a, s])
            raw[s, b] += c * int(dsrv[s, b])
    return (raw + raw.T) / 2.0 / n_tokens, raw


@nb.njit(cache=True, parallel=True)
def _fused_pass(sel, packed, P, bounds, t0, E, nblk):
    N, L, K = sel.shape
    C = bounds.shape[0] - 1
    G = packed.shape[0]
    cnt = np.zeros((nblk, L, E), dtype=np.int32)
    sums = np.zeros((nblk, 4 * G, C), dtype=np.int64)
    step = (N + nblk - 1) // nblk
    for b in nb.prange(nblk):
        lo = b * step
        hi = min(N, lo + step)
        if lo >= hi:
            continue
        acc = np.zeros(4 * G, dtype=np.int64)
        c = np.searchsorted(bounds, lo + t0, side="right") - 1
        for t in range(lo, hi):
            while bounds[c + 1] <= t + t0:
                for q in range(4 * G):
                    sums[b, q, c] += acc[q]
                    acc[q] = 0
                c += 1
            for l in range(L):
                for k in range(K):
                    cnt[b, l, sel[t, l, k]] += 1
                for g in range(G):
                    w = np.uint64(0)
                    for k in range(K):
                        w += packed[g, l, sel[t, l, k]]
                    acc[4 * g] += np.int64(w & np.uint64(0xFFFF))
                    acc[4 * g + 1] += np.int64((w >> np.uint64(16)) & np.uint64(0xFFFF))
                    acc[4 * g + 2] += np.int64((w >> np.uint64(32)) & np.uint64(0xFFFF))
                    acc[4 * g + 3] += np.int64(w >> np.uint64(48))
        for q in range(4 * G):
            sums[b, q, c] += acc[q]
    out = np.zeros((L, E), dtype=np.int64)
    for b in range(nblk):
        out += cnt[b]
    return out, sums.sum(axis=0)


def fused_pass(sel, pes, bounds, E: int, t0: int = 0, blocks: int = 0):
    """One pass over the trace: counts [L, E] and per-chunk hop sums [P, C] of every placement —
    the CPU baseline's best form: token blocks in parallel with private partials and an integer
    merge, and the P placements' per-expert costs packed four 16-bit lanes to a 64-bit word so a
    pick costs one table gather per 4 placements (per-layer lane sums <= K*255 < 2^16)."""
    sel = np.ascontiguousarray(sel)
    pes = [np.asarray(x, dtype=np.int64) for x in pes]
    P = len(pes)
    L, Ee = pes[0].shape
    if K_max_ok(sel.shape[2], max(int(x.max(initial=0)) for x in pes)) is False:
        raise ValueError("per-layer lane sum would overflow 16 bits")
    G = (P + 3) // 4
    packed = np.zeros((G, L, E), dtype=np.uint64)
    for q, x in enumerate(pes):
        packed[q // 4, :, :Ee] |= x.astype(np.uint64) << np.uint64(16 * (q % 4))
    nblk = blocks or nb.get_num_threads()  # one private partial per thread: merge cost O(threads*L*E)
    cnt, sums = _fused_pass(sel, packed, P, np.asarray(bounds, dtype=np.int64), np.int64(t0), E,
                            max(1, min(nblk, sel.shape[0])))
    return cnt, sums[:P]


def K_max_ok(K: int, max_p: int) -> bool:
    return K * max_p < (1 << 16)


@nb.njit(cache=True, parallel=True)
def _dedup_sums(sel, pe, srv_e, src, bounds, t0):
    C = bounds.shape[0] - 1
    N, L, K = sel.shape
    hop = np.zeros(C, dtype=np.int64)
    uq = np.zeros(C, dtype=np.int64)
    dd = np.zeros(C, dtype=np.int64)
    for c in nb.prange(C):
        lo = max(bounds[c], t0) - t0
        hi = min(bounds[c + 1], t0 + N) - t0
        h = 0
        u = 0
        d = 0
        for t in range(lo, hi):
            for l in range(L):
                seen = np.empty(K, dtype=np.int64)
                ns = 0
                for k in range(K):
                    e = sel[t, l, k]
                    s = srv_e[l, e]
                    h += pe[l, e]
                    new = True
                    for j in range(ns):
                        if seen[j] == s:
                            new = False
                    if new:
                        seen[ns] = s
                        ns += 1
                        d += pe[l, e]
                        if s != src[l]:
                            u += 1
        hop[c] = h
        uq[c] = u
        dd[c] = d
    return hop, uq, dd


def dedup_sums(sel, pe, srv_e, src, bounds, t0: int = 0):
    """Extension A17 restated: per chunk (SPEC hops, unique remote destination servers,
    hops with one message per destination server).  srv_e[l, e] = server hosting expert e,
    src[l] = dispatch server of layer l."""
    return _dedup_sums(np.ascontiguousarray(sel), np.ascontiguousarray(pe, dtype=np.int64),
                       np.ascontiguousarray(srv_e, dtype=np.int64), np.asarray(src, dtype=np.int64),
                       np.asarray(bounds, dtype=np.int64), np.int64(t0))
