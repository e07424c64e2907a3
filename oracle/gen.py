"""Oracle trace generator (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

SPEC.md:123-131, 166 define the law: per layer an independent random permutation maps expert
ranks to a Zipf(s) popularity; each token draws K experts without replacement proportionally to
popularity; deterministic given the seed; tokens evenly labelled into chunks.  The concrete
sampler (ours, shared by the GPU kernel so shards regenerate bit-identically):
  * weights w_r = max(1, floor(2^30 * r^-s / sum_j j^-s)), r = 1..E; cdf = prefix sums;
  * permutation: Fisher-Yates, j = floor(u * (i+1) / 2^32), u = Philox4x32-10(i, 0, l, 2^30).x;
  * draw k of (t, l): u = Philox4x32-10(t_lo, t_hi, l, k // 4)[k % 4]; x = floor(u * W_rem / 2^32)
    over the weight line with chosen rank intervals removed; rank = last r with cdf[r] <= x;
  * chunk(t) = floor(t * C / N).
"""
from __future__ import annotations

import numba as nb
import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


@nb.njit(cache=True, inline="always")
def philox(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11) on python-int-like uint64 values."""
    for _ in range(10):
        p0 = np.uint64(M0) * np.uint64(c0)
        p1 = np.uint64(M1) * np.uint64(c2)
        hi0 = (p0 >> np.uint64(32)) & np.uint64(MASK)
        lo0 = p0 & np.uint64(MASK)
        hi1 = (p1 >> np.uint64(32)) & np.uint64(MASK)
        lo1 = p1 & np.uint64(MASK)
        n0 = hi1 ^ np.uint64(c1) ^ np.uint64(k0)
        n2 = hi0 ^ np.uint64(c3) ^ np.uint64(k1)
        c0, c1, c2, c3 = n0, lo1, n2, lo0
        k0 = (np.uint64(k0) + np.uint64(W0)) & np.uint64(MASK)
        k1 = (np.uint64(k1) + np.uint64(W1)) & np.uint64(MASK)
    return np.uint64(c0), np.uint64(c1), np.uint64(c2), np.uint64(c3)


def weights(E: int, s: float) -> np.ndarray:
    r = np.arange(1, E + 1, dtype=np.float64)
    raw = r ** (-float(s))
    return np.maximum(1, np.floor(raw / raw.sum() * (1 << 30))).astype(np.int64)


def cdf(E: int, s: float) -> np.ndarray:
    return np.concatenate([[0], np.cumsum(weights(E, s))]).astype(np.int64)


@nb.njit(cache=True)
def _perms(seed, L, E):
    k0 = np.uint64(seed & MASK)
    k1 = np.uint64((seed >> 32) & MASK)
    out = np.empty((L, E), dtype=np.int64)
    for l in range(L):
        p = np.arange(E)
        for i in range(E - 1, 0, -1):
            u, _, _, _ = philox(np.uint64(i), np.uint64(0), np.uint64(l), np.uint64(0x40000000), k0, k1)
            j = (u * np.uint64(i + 1)) >> np.uint64(32)
            jj = np.int64(j)
            tmp = p[i]
            p[i] = p[jj]
            p[jj] = tmp
        out[l] = p
    return out


def perms(seed: int, L: int, E: int) -> np.ndarray:
    return _perms(np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), L, E)


@nb.njit(cache=True, parallel=True)
def _generate(seed, t0, n, L, K, E, cdf_, perm):
    k0 = np.uint64(seed & MASK)
    k1 = np.uint64((seed >> 32) & MASK)
    out = np.empty((n, L, K), dtype=np.uint8)
    total = cdf_[E]
    for i in nb.prange(n):
        t = np.uint64(t0 + i)
        t_lo = t & np.uint64(MASK)
        t_hi = t >> np.uint64(32)
        ch = np.empty(K, dtype=np.int64)
        for l in range(L):
            nch = 0
            rem = total
            r0 = r1 = r2 = r3 = np.uint64(0)
            for k in range(K):
                if k % 4 == 0:
                    r0, r1, r2, r3 = philox(t_lo, t_hi, np.uint64(l), np.uint64(k // 4), k0, k1)
                q = k % 4
                u = r0 if q == 0 else (r1 if q == 1 else (r2 if q == 2 else r3))
                x = np.int64((u * np.uint64(rem)) >> np.uint64(32))
                for j in range(nch):
                    c = ch[j]
                    if cdf_[c] <= x:
                        x += cdf_[c + 1] - cdf_[c]
                    else:
                        break
                r = np.searchsorted(cdf_, x, side="right") - 1
                j = nch
                while j > 0 and ch[j - 1] > r:
                    ch[j] = ch[j - 1]
                    j -= 1
                ch[j] = r
                nch += 1
                rem -= cdf_[r + 1] - cdf_[r]
                out[i, l, k] = perm[l, r]
    return out


def generate(L: int, E: int, K: int, zipf_s: float, n_tokens: int, n_chunks: int, seed: int,
             tok_range=None):
    """Token-major uint8 [n, L, K] selections of tokens [a, b) plus the full chunk bounds."""
    a, b = (0, n_tokens) if tok_range is None else tok_range
    c = cdf(E, zipf_s)
    p = perms(seed, L, E)
    sel = _generate(np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), np.int64(a), np.int64(b - a), L, K, E, c, p)
    bounds = np.array([(ci * n_tokens + n_chunks - 1) // n_chunks for ci in range(n_chunks + 1)], dtype=np.int64)
    return sel, bounds
