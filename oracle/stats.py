"""Oracle load statistics (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

estimate_frequencies: count(l, e) over every (token, pick); f = count/(K*N).
Parallel over token blocks with per-block private counts and an order-independent integer merge
(SPEC.md:168), so the result is independent of the thread count.
"""
from __future__ import annotations

import numba as nb
import numpy as np


@nb.njit(cache=True, parallel=True)
def _counts(sel, E, nblk):
    N, L, K = sel.shape
    part = np.zeros((nblk, L, E), dtype=np.int64)
    step = (N + nblk - 1) // nblk
    for b in nb.prange(nblk):
        lo = b * step
        hi = min(N, lo + step)
        for t in range(lo, hi):
            for l in range(L):
                for k in range(K):
                    part[b, l, sel[t, l, k]] += 1
    return part.sum(axis=0)


def counts(sel: np.ndarray, E: int, blocks: int = 0) -> np.ndarray:
    """int64 [L, E] selection counts of token-major uint8 selections [N, L, K]."""
    sel = np.ascontiguousarray(sel)
    if sel.shape[0] == 0:
        return np.zeros((sel.shape[1], E), dtype=np.int64)
    if sel.max(initial=0) >= E:
        raise ValueError("expert index >= E")
    return _counts(sel, E, max(1, min(blocks or nb.get_num_threads(), sel.shape[0])))


def counts_bincount(sel: np.ndarray, E: int) -> np.ndarray:
    """Independent cross-check: numpy.bincount per layer."""
    N, L, K = sel.shape
    return np.stack([np.bincount(sel[:, l, :].ravel(), minlength=E) for l in range(L)]).astype(np.int64)


def frequencies(cnt: np.ndarray, n_tokens: int, K: int) -> np.ndarray:
    if n_tokens == 0:
        raise ValueError("empty trace")
    return cnt / (K * n_tokens)
