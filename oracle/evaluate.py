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
