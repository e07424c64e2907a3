"""``moeplace.topology`` — cluster graphs, the hop-distance matrix and the locality ordering
(SPEC.md:17-89).

``build_topology`` and ``locality_order`` are host code (small graphs).
``all_pairs_hops`` runs the BFS on the GPU (``mp_apsp_bfs``, one CTA per source server) and keeps
the server-level hop matrix resident on the device, where ``cost_matrix`` consumes it.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _lib
from .errors import ConfigError, TopologyError

KINDS = ("FatTree", "FatTreeHier", "Dragonfly", "DragonflySparse")
EXTENSION_KINDS = ("DragonflyPlus", "SlimFly")  # not in SPEC; graph-only extensions


@dataclass(frozen=True)
class TopologySpec:
    """SPEC.md:22-27.  ``extra`` holds kind-specific parameters:
    FatTree ``spines`` (default 4); FatTreeHier ``groups`` (default 4); Dragonfly
    ``group_size`` (default 4); DragonflyPlus ``group_size`` (4) and ``spines_per_group`` (2)."""

    kind: str
    num_leaf_switches: int
    servers_per_leaf: int
    gpus_per_server: int
    extra: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.kind not in KINDS + EXTENSION_KINDS:
            raise ConfigError(f"unknown topology kind {self.kind!r}; expected one of {KINDS + EXTENSION_KINDS}")
        for name in ("num_leaf_switches", "servers_per_leaf", "gpus_per_server"):
            v = getattr(self, name)
            if not isinstance(v, (int, np.integer)) or v < 1:
                raise ConfigError(f"TopologySpec.{name} must be an integer >= 1, got {v!r}")

    @property
    def n_servers(self) -> int:
        return self.num_leaf_switches * self.servers_per_leaf

    @property
    def n_devices(self) -> int:
        return self.n_servers * self.gpus_per_server

    def to_json(self) -> dict:
        return {"kind": self.kind, "num_leaf_switches": int(self.num_leaf_switches),
                "servers_per_leaf": int(self.servers_per_leaf), "gpus_per_server": int(self.gpus_per_server),
                "extra": dict(self.extra)}


@dataclass
class ClusterGraph:
    """SPEC.md:28-33.  Node ids: servers are 0..n_servers-1, switches follow.  Devices are not
    graph nodes (intra-server distance is 0 by convention); ``device_server[d]`` owns device d."""

    spec: TopologySpec
    device_server: np.ndarray   # int32 [S]
    server_leaf: np.ndarray     # int32 [n_servers], node id of the leaf switch
    switch_kind: list           # kind of node n_servers + i: leaf/spine/aggregation/top
    links: np.ndarray           # int32 [n_links, 2], undirected, a < b

    @property
    def n_servers(self) -> int:
        return int(self.server_leaf.shape[0])

    @property
    def n_devices(self) -> int:
        return int(self.device_server.shape[0])

    @property
    def n_nodes(self) -> int:
        return self.n_servers + len(self.switch_kind)

    @property
    def leaf_nodes(self) -> np.ndarray:
        return np.array([self.n_servers + i for i, k in enumerate(self.switch_kind) if k == "leaf"], dtype=np.int32)

    def csr(self) -> tuple[np.ndarray, np.ndarray]:
        """Symmetric CSR adjacency (row_ptr int32[n+1], col int32[2*n_links]); neighbours ascending."""
        n = self.n_nodes
        a = np.concatenate([self.links[:, 0], self.links[:, 1]]).astype(np.int64)
        b = np.concatenate([self.links[:, 1], self.links[:, 0]]).astype(np.int64)
        order = np.lexsort((b, a))
        a, b = a[order], b[order]
        row_ptr = np.zeros(n + 1, dtype=np.int32)
        np.add.at(row_ptr, a + 1, 1)
        row_ptr = np.cumsum(row_ptr).astype(np.int32)
        return row_ptr, b.astype(np.int32)

    def to_json(self) -> dict:
        """Export document {spec, nodes:[{id,kind,parent}], links:[[a,b]]}.  Device d
        is exported as node id ``n_nodes + d`` with its server as parent."""
        nodes = []
        for s in range(self.n_servers):
            nodes.append({"id": s, "kind": "server", "parent": int(self.server_leaf[s])})
        for i, k in enumerate(self.switch_kind):
            nodes.append({"id": self.n_servers + i, "kind": k, "parent": None})
        for d in range(self.n_devices):
            nodes.append({"id": self.n_nodes + d, "kind": "device", "parent": int(self.device_server[d])})
        return {"spec": self.spec.to_json(), "nodes": nodes, "links": self.links.tolist()}

    @classmethod
    def from_json(cls, doc: dict) -> "ClusterGraph":
        try:
            s = doc["spec"]
            spec = TopologySpec(s["kind"], s["num_leaf_switches"], s["servers_per_leaf"], s["gpus_per_server"],
                                dict(s.get("extra", {})))
            servers = sorted((n for n in doc["nodes"] if n["kind"] == "server"), key=lambda n: n["id"])
            switches = sorted((n for n in doc["nodes"] if n["kind"] not in ("server", "device")), key=lambda n: n["id"])
            devices = sorted((n for n in doc["nodes"] if n["kind"] == "device"), key=lambda n: n["id"])
        except (KeyError, TypeError) as e:
            raise TopologyError(f"malformed topology document: {e}") from None
        links = np.array(doc["links"], dtype=np.int32).reshape(-1, 2)
        return cls(spec, np.array([d["parent"] for d in devices], dtype=np.int32),
                   np.array([n["parent"] for n in servers], dtype=np.int32), [n["kind"] for n in switches], links)


class _Builder:
    def __init__(self, spec: TopologySpec):
        self.spec = spec
        self.n_srv = spec.n_servers
        self.kinds: list[str] = []
        self.edges: set[tuple[int, int]] = set()

    def switch(self, kind: str) -> int:
        self.kinds.append(kind)
        return self.n_srv + len(self.kinds) - 1

    def link(self, a: int, b: int):
        if a != b:
            self.edges.add((min(a, b), max(a, b)))

    def done(self, leaves: list[int]) -> ClusterGraph:
        spec = self.spec
        server_leaf = np.repeat(np.array(leaves, dtype=np.int32), spec.servers_per_leaf)
        for s in range(self.n_srv):
            self.link(s, int(server_leaf[s]))
        device_server = np.repeat(np.arange(self.n_srv, dtype=np.int32), spec.gpus_per_server)
        links = np.array(sorted(self.edges), dtype=np.int32).reshape(-1, 2)
        return ClusterGraph(spec, device_server, server_leaf, list(self.kinds), links)


def _xparam(spec: TopologySpec, name: str, default: int) -> int:
    v = spec.extra.get(name, default)
    if not isinstance(v, (int, np.integer)) or v < 1:
        raise ConfigError(f"{spec.kind} parameter {name!r} must be an integer >= 1, got {v!r}")
    return int(v)


def build_topology(spec: TopologySpec) -> ClusterGraph:
    """SPEC.md:42-50 with the wiring fixed at SPEC.md:77.  Leaves are numbered 0..n-1 and leaf i
    owns servers i*spl .. i*spl+spl-1; devices of server s are s*gps .. s*gps+gps-1."""
    n = spec.num_leaf_switches
    b = _Builder(spec)
    leaves = [b.switch("leaf") for _ in range(n)]
    kind = spec.kind
    if kind == "FatTree":
        spines = [b.switch("spine") for _ in range(_xparam(spec, "spines", 4))]
        for lf in leaves:
            for sp in spines:
                b.link(lf, sp)
    elif kind == "FatTreeHier":
        groups = min(_xparam(spec, "groups", 4), n)
        aggs = [b.switch("aggregation") for _ in range(groups)]
        top = b.switch("top")
        for i, lf in enumerate(leaves):
            b.link(lf, aggs[i * groups // n])
        for a in aggs:
            b.link(a, top)
    elif kind == "Dragonfly":
        gs = _xparam(spec, "group_size", 4)
        ngroups = (n + gs - 1) // gs
        members = [leaves[g * gs:(g + 1) * gs] for g in range(ngroups)]
        for grp in members:
            for i in range(len(grp)):
                for j in range(i + 1, len(grp)):
                    b.link(grp[i], grp[j])
        rr = [0] * ngroups  # round-robin endpoint choice per group
        for g in range(ngroups):
            for h in range(g + 1, ngroups):
                a = members[g][rr[g] % len(members[g])]
                c = members[h][rr[h] % len(members[h])]
                rr[g] += 1
                rr[h] += 1
                b.link(a, c)
    elif kind == "DragonflySparse":
        if n == 2:
            raise ConfigError("DragonflySparse needs >= 3 leaf switches for the diameter chord (or exactly 1)")
        for i in range(n):
            b.link(leaves[i], leaves[(i + 1) % n])
            b.link(leaves[i], leaves[(i + n // 2) % n])
    elif kind == "DragonflyPlus":
        gs = _xparam(spec, "group_size", 4)
        nsp = _xparam(spec, "spines_per_group", 2)
        ngroups = (n + gs - 1) // gs
        gspines = []
        for g in range(ngroups):
            sps = [b.switch("spine") for _ in range(nsp)]
            gspines.append(sps)
            for lf in leaves[g * gs:(g + 1) * gs]:
                for sp in sps:
                    b.link(lf, sp)
        rr = [0] * ngroups
        for g in range(ngroups):
            for h in range(g + 1, ngroups):
                b.link(gspines[g][rr[g] % nsp], gspines[h][rr[h] % nsp])
                rr[g] += 1
                rr[h] += 1
    elif kind == "SlimFly":
        _slimfly_links(b, leaves)
    else:  # pragma: no cover - rejected by TopologySpec
        raise ConfigError(kind)
    return b.done(leaves)


def _slimfly_links(b: _Builder, leaves: list[int]):
    """McKay-Miller-Siran graph over 2*q^2 routers (q prime, q = 4w + 1 or 4w - 1), the Slim Fly
    router graph (diameter 2).  Leaves are the routers."""
    n = len(leaves)
    q = int(round((n / 2) ** 0.5))
    if 2 * q * q != n or q < 3 or any(q % d == 0 for d in range(2, int(q ** 0.5) + 1)) or q % 4 == 2:
        raise ConfigError("SlimFly needs num_leaf_switches = 2*q^2 with q an odd prime (e.g. 18, 50, 98)")
    xi = next(g for g in range(2, q) if len({pow(g, k, q) for k in range(1, q)}) == q - 1)  # primitive root
    d = 1 if q % 4 == 1 else -1
    w = (q - d) // 4
    if q % 4 == 1:
        X = {pow(xi, k, q) for k in range(0, q - 1, 2)}
        Xp = {pow(xi, k, q) for k in range(1, q - 1, 2)}
    else:
        X = {pow(xi, k, q) for k in list(range(0, 2 * w - 1, 2)) + list(range(2 * w - 1, 4 * w - 2, 2))}
        Xp = {pow(xi, k, q) for k in list(range(1, 2 * w, 2)) + list(range(2 * w, 4 * w - 1, 2))}

    def r0(x, y):
        return leaves[x * q + y]

    def r1(m, c):
        return leaves[q * q + m * q + c]

    for x in range(q):
        for y in range(q):
            for yp in range(q):
                if (y - yp) % q in X:
                    b.link(r0(x, y), r0(x, yp))
    for m in range(q):
        for c in range(q):
            for cp in range(q):
                if (c - cp) % q in Xp:
                    b.link(r1(m, c), r1(m, cp))
    for x in range(q):
        for y in range(q):
            for m in range(q):
                b.link(r0(x, y), r1(m, (m * x + y) % q))


@dataclass
class DistanceMatrix:
    """SPEC.md:34-39.  Hop counts are stored at server granularity on the device
    (``server_dist``: uint8 [n_servers, n_servers]); device-level entries are
    ``dist(u, v) = server_dist[server(u), server(v)]`` (0 on the same server)."""

    graph: ClusterGraph
    server_dist: Any            # torch.uint8 [n_srv, n_srv], CUDA
    _dev: Any = None

    @property
    def n_devices(self) -> int:
        return self.graph.n_devices

    @property
    def dist(self):
        """Device-level matrix, torch.uint8 [S, S] on the GPU (expanded by ``mp_expand_dist``)."""
        if self._dev is None:
            t = _lib.torch()
            g = self.graph
            S = g.n_devices
            out = t.empty((S, S), dtype=t.uint8, device=self.server_dist.device)
            srv = _lib.to_dev(g.device_server, t.int32)
            _lib.call("mp_expand_dist", _lib.ptr(self.server_dist), g.n_servers, _lib.ptr(srv), S, _lib.ptr(out),
                      _lib.stream_handle())
            self._dev = out
        return self._dev

    def numpy(self) -> np.ndarray:
        return self.dist.cpu().numpy()

    def server_numpy(self) -> np.ndarray:
        return self.server_dist.cpu().numpy()

    def to_csv(self, path) -> None:
        """Square CSV, header row = device ids."""
        d = self.numpy()
        S = d.shape[0]
        with open(path, "w") as f:
            f.write(",".join(str(i) for i in range(S)) + "\n")
            for r in range(S):
                f.write(",".join(str(int(v)) for v in d[r]) + "\n")


def all_pairs_hops(g: ClusterGraph) -> DistanceMatrix:
    """SPEC.md:51-59.  BFS from every server over the unit-weight switch graph, on the GPU."""
    t = _lib.torch()
    _lib.require_cuda()
    row_ptr, col = g.csr()
    srv = np.arange(g.n_servers, dtype=np.int32)
    d_row, d_col, d_srv = (_lib.to_dev(row_ptr, t.int32), _lib.to_dev(col if col.size else np.zeros(1, np.int32), t.int32),
                           _lib.to_dev(srv, t.int32))
    out = t.empty((g.n_servers, g.n_servers), dtype=t.uint8, device=d_srv.device)
    err = _lib.new_err()
    _lib.call("mp_apsp_bfs", _lib.ptr(d_row), _lib.ptr(d_col), g.n_nodes, _lib.ptr(d_srv), g.n_servers,
              _lib.ptr(d_srv), g.n_servers, _lib.ptr(out), _lib.ptr(err), _lib.stream_handle())
    code, a, b, n = _lib.read_err(err)
    if code == _lib.DATA_UNREACHABLE:
        raise TopologyError(f"graph is disconnected: server {b} unreachable from server {a} ({n} pairs)")
    if code == _lib.DATA_HOPS_RANGE:
        raise ConfigError(f"hop count between servers {a} and {b} exceeds 255 (u8 device format)")
    if code:
        raise TopologyError(f"BFS error code {code}")
    return DistanceMatrix(g, out)


def locality_order(g: ClusterGraph, d: DistanceMatrix) -> list[int]:
    """devices of a server contiguous, servers of a leaf contiguous, leaves in a
    nearest-neighbour tour over leaf-to-leaf distances starting at leaf 0 (ties: lowest id)."""
    D = d.server_numpy().astype(np.int64)
    spl = g.spec.servers_per_leaf
    n_leaf = g.n_servers // spl
    first = np.arange(n_leaf) * spl
    LD = D[np.ix_(first, first)]  # leaf-to-leaf via their first servers (same +2 offset everywhere)
    seen = np.zeros(n_leaf, dtype=bool)
    cur, tour = 0, [0]
    seen[0] = True
    for _ in range(n_leaf - 1):
        cand = np.where(~seen)[0]
        nxt = int(cand[np.argmin(LD[cur, cand])])  # argmin returns the lowest index on ties
        seen[nxt] = True
        tour.append(nxt)
        cur = nxt
    gps = g.spec.gpus_per_server
    order = []
    for leaf in tour:
        for s in range(leaf * spl, (leaf + 1) * spl):
            order.extend(range(s * gps, (s + 1) * gps))
    return order


def save_topology(g: ClusterGraph, path) -> None:
    with open(path, "w") as f:
        json.dump(g.to_json(), f)


def load_topology(path) -> ClusterGraph:
    with open(path) as f:
        return ClusterGraph.from_json(json.load(f))
