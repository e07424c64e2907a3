"""Oracle hop matrix, cost matrix and ILP coefficients (TEST INFRASTRUCTURE ONLY).

all_pairs_hops: unit-weight BFS over the {server, switch} graph from every
server; 0 on the same server; a disconnected graph is an error.
cost_matrix: p[l, s] = D(d_l, s) + D(s, c_l).
build_instance: w = f[:, :, None] * p[:, None, :], w_int = rint(w * 1e9).
"""
from __future__ import annotations

from collections import deque

import numpy as np


def bfs_apsp(n_nodes: int, links, sources) -> np.ndarray:
    """int64 [len(sources), n_nodes] hop counts (-1 = unreachable)."""
    adj = [[] for _ in range(n_nodes)]
    for a, b in links:
        adj[int(a)].append(int(b))
        adj[int(b)].append(int(a))
    out = np.full((len(sources), n_nodes), -1, dtype=np.int64)
    for i, s in enumerate(sources):
        d = out[i]
        d[s] = 0
        q = deque([s])
        while q:
            u = q.popleft()
            for v in adj[u]:
                if d[v] < 0:
                    d[v] = d[u] + 1
                    q.append(v)
    return out


def server_hops(n_nodes: int, links, n_servers: int) -> np.ndarray:
    """Server x server hops; raises ValueError if some server is unreachable."""
    d = bfs_apsp(n_nodes, links, list(range(n_servers)))[:, :n_servers]
    if (d < 0).any():
        raise ValueError("disconnected graph")
    return d


def device_hops(dsrv: np.ndarray, device_server: np.ndarray) -> np.ndarray:
    return dsrv[np.ix_(device_server, device_server)]


def cost_matrix(dsrv: np.ndarray, device_server: np.ndarray, dispatch, collect) -> np.ndarray:
    D = device_hops(dsrv, device_server)
    d = np.asarray(dispatch)
    c = np.asarray(collect)
    return (D[d, :] + D[:, c].T).astype(np.int64)


def coefficients(f: np.ndarray, p: np.ndarray, scale: float = 1e9):
    w = f[:, :, None] * p.astype(np.float64)[:, None, :]
    return w, np.rint(w * scale).astype(np.int64)
