"""``moeplace.placement`` — constraints, placements, the cost matrix and the two heuristic
placers.

``cost_matrix`` runs on the GPU (``mp_cost_matrix``) and stays device resident for the scorer.
``validate``, ``place_round_robin`` and ``place_greedy`` are sequential host algorithms by
definition and are not on the data-parallel path.
"""
from __future__ import annotations

import csv
from dataclasses import dataclass
from typing import Any, Optional, Sequence

import numpy as np

from . import _lib
from .errors import ConfigError, InfeasibleError, MoeplaceError, TraceParseError
from .model_trace import AttentionPlacement, ModelSpec
from .topology import DistanceMatrix


@dataclass(frozen=True)
class Constraints:
    """C^exp experts per device, C^layer experts per (device, layer)."""

    c_exp: int
    c_layer: int

    def __post_init__(self):
        if self.c_layer < 1 or self.c_exp < self.c_layer:
            raise ConfigError(f"need c_layer >= 1 and c_exp >= c_layer, got c_exp={self.c_exp}, c_layer={self.c_layer}")

    def check_feasible(self, model: ModelSpec, n_devices: int) -> None:
        """S*c_exp >= L*E and S*c_layer >= E."""
        if n_devices * self.c_exp < model.L * model.E:
            raise InfeasibleError(f"capacity: {n_devices} devices x c_exp={self.c_exp} < L*E={model.L * model.E}")
        if n_devices * self.c_layer < model.E:
            raise InfeasibleError(f"capacity: {n_devices} devices x c_layer={self.c_layer} < E={model.E}")


@dataclass
class Placement:
    """assign[l, e] = device of expert e of layer l (y_{les} in one-hot form)."""

    assign: np.ndarray  # int32 [L, E]
    constraints: Optional[Constraints] = None
    label: str = ""

    def __post_init__(self):
        self.assign = np.ascontiguousarray(self.assign, dtype=np.int32)
        if self.assign.ndim != 2:
            raise ConfigError("Placement.assign must be a 2-D [L, E] array")


@dataclass
class CostMatrix:
    """p[l, s] = dist(d_l, s) + dist(s, c_l), uint8 [L, S] on the device."""

    p: Any                              # torch.uint8 [L, S] (CUDA)
    dist: Optional[DistanceMatrix] = None
    attn: Optional[AttentionPlacement] = None

    @property
    def L(self) -> int:
        return int(self.p.shape[0])

    @property
    def S(self) -> int:
        return int(self.p.shape[1])

    def numpy(self) -> np.ndarray:
        return self.p.cpu().numpy()

    @property
    def max_p(self) -> int:
        return int(self.p.max().item()) if self.p.numel() else 0


@dataclass
class Violation:
    """One violated constraint of Eq. (1)."""

    family: str                 # "assignment" | "c_layer" | "c_exp"
    layer: Optional[int]
    expert: Optional[int]
    device: Optional[int]
    count: int = 0
    limit: int = 0


def cost_matrix(dist: DistanceMatrix, attn: AttentionPlacement) -> CostMatrix:
    """SPEC.md:198-206, computed on the GPU from the server-level hop matrix."""
    t = _lib.torch()
    g = dist.graph
    S, L = g.n_devices, int(attn.dispatch.shape[0])
    if attn.dispatch.min(initial=0) < 0 or max(attn.dispatch.max(initial=0), attn.collect.max(initial=0)) >= S \
            or attn.collect.min(initial=0) < 0:
        raise ConfigError("attention placement refers to a device outside the topology")
    dmax = int(dist.server_dist.max().item()) if dist.server_dist.numel() else 0
    if 2 * dmax > 255:
        raise ConfigError(f"round-trip hop cost 2*{dmax} exceeds 255 (u8 device format)")
    p = t.empty((L, S), dtype=t.uint8, device=dist.server_dist.device)
    srv = _lib.to_dev(g.device_server, t.int32)
    d = _lib.to_dev(attn.dispatch, t.int32)
    c = _lib.to_dev(attn.collect, t.int32)
    _lib.call("mp_cost_matrix", _lib.ptr(dist.server_dist), g.n_servers, _lib.ptr(srv), S, _lib.ptr(d), _lib.ptr(c), L,
              _lib.ptr(p), _lib.stream_handle())
    return CostMatrix(p, dist, attn)


def validate(p: Placement, c: Constraints, model: ModelSpec, n_devices: int) -> list[Violation]:
    """Every violated constraint; an empty list means the placement is feasible."""
    a = p.assign
    out: list[Violation] = []
    if a.shape != (model.L, model.E):
        return [Violation("assignment", None, None, None, int(a.size), model.L * model.E)]
    bad = np.argwhere((a < 0) | (a >= n_devices))
    for l, e in bad:
        out.append(Violation("assignment", int(l), int(e), int(a[l, e]), 0, 1))
    ok = (a >= 0) & (a < n_devices)
    per_layer = np.zeros((model.L, n_devices), dtype=np.int64)
    rows = np.repeat(np.arange(model.L), model.E).reshape(model.L, model.E)
    np.add.at(per_layer, (rows[ok], a[ok]), 1)
    for l, s in np.argwhere(per_layer > c.c_layer):
        out.append(Violation("c_layer", int(l), None, int(s), int(per_layer[l, s]), c.c_layer))
    total = per_layer.sum(axis=0)
    for s in np.where(total > c.c_exp)[0]:
        out.append(Violation("c_exp", None, None, int(s), int(total[s]), c.c_exp))
    return out


def place_round_robin(model: ModelSpec, attn: AttentionPlacement, order: Sequence[int], c: Constraints) -> Placement:
    """SPEC.md:216-224.  d = ceil(E / c_layer); layer l with dispatch at ordering position i uses
    the circular window [i - floor(d/2), i + ceil(d/2)); expert e goes to window slot
    floor(e / c_layer).  (The stated formula is followed where SPEC.md:222's prose differs.)"""
    order = np.asarray(list(order), dtype=np.int64)
    n = order.shape[0]
    pos = np.full(int(order.max(initial=-1)) + 1, -1, dtype=np.int64)
    pos[order] = np.arange(n)
    L, E = model.L, model.E
    d = -(-E // c.c_layer)
    if d > n:
        raise InfeasibleError(f"round robin window d={d} exceeds {n} devices")
    slots = np.arange(E) // c.c_layer
    assign = np.empty((L, E), dtype=np.int32)
    used = np.zeros(max(n, int(order.max(initial=0)) + 1), dtype=np.int64)
    for l in range(L):
        dl = int(attn.dispatch[l])
        if dl >= pos.shape[0] or pos[dl] < 0:
            raise ConfigError(f"dispatch device {dl} of layer {l} is not in the ordering")
        i = int(pos[dl])
        devs = order[(i - d // 2 + slots) % n]
        assign[l] = devs
        np.add.at(used, devs, 1)
        over = np.where(used[devs] > c.c_exp)[0]
        if over.size:
            s = int(devs[over[0]])
            raise InfeasibleError(f"round robin: device {s} exceeds c_exp={c.c_exp} at layer {l}")
    return Placement(assign, c, "rr")


def place_greedy(model: ModelSpec, attn: AttentionPlacement, cost: CostMatrix, c: Constraints) -> Placement:
    """layers 0..L-1, experts 0..E-1, each to the first device in
    p[l, .]-ascending order (ties: lower id) with residual c_layer and c_exp capacity."""
    p = cost.numpy().astype(np.int64)
    L, S = p.shape
    E = model.E
    used = np.zeros(S, dtype=np.int64)
    assign = np.empty((L, E), dtype=np.int32)
    for l in range(L):
        order = np.lexsort((np.arange(S), p[l]))
        layer_used = np.zeros(S, dtype=np.int64)
        k = 0
        for e in range(E):
            # devices before k are full for this layer (capacities only shrink): skip them once
            while k < S and (layer_used[order[k]] >= c.c_layer or used[order[k]] >= c.c_exp):
                k += 1
            if k == S:
                raise InfeasibleError(f"greedy: no feasible device for expert ({l}, {e})")
            s = int(order[k])
            assign[l, e] = s
            layer_used[s] += 1
            used[s] += 1
    return Placement(assign, c, "greedy")


def perturb_swaps(p: Placement, n_candidates: int, n_swaps: int, seed0: int = 1000) -> np.ndarray:
    """Candidate placements for batched scoring (BASELINE config 4): candidate i applies
    ``n_swaps`` within-layer swaps drawn with seed ``seed0 + i`` to ``p``.  Swapping the devices of
    two experts of the same layer keeps every per-(device, layer) and per-device count, so all
    candidates satisfy the constraints ``p`` satisfies.  Returns int32 [n_candidates, L, E]."""
    L, E = p.assign.shape
    out = np.repeat(p.assign[None], n_candidates, axis=0).astype(np.int32)
    for i in range(n_candidates):
        rng = np.random.default_rng(seed0 + i)
        ls = rng.integers(0, L, n_swaps)
        a = rng.integers(0, E, n_swaps)
        b = rng.integers(0, E, n_swaps)
        c = out[i]
        for l, x, y in zip(ls, a, b):
            c[l, x], c[l, y] = c[l, y], c[l, x]
    return out


def write_placement(p: Placement, path) -> None:
    """CSV with header layer,expert,device."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(["layer", "expert", "device"])
        L, E = p.assign.shape
        for l in range(L):
            for e in range(E):
                w.writerow([l, e, int(p.assign[l, e])])


def read_placement(path, model: ModelSpec, c: Optional[Constraints] = None, n_devices: Optional[int] = None) -> Placement:
    """Load a placement CSV; re-validates when constraints are given."""
    assign = np.full((model.L, model.E), -1, dtype=np.int32)
    with open(path, newline="") as f:
        r = csv.reader(f)
        header = next(r, None)
        if header != ["layer", "expert", "device"]:
            raise ConfigError(f"{path}: expected header layer,expert,device")
        for ln, row in enumerate(r, start=2):
            try:
                l, e, s = (int(v) for v in row)
            except ValueError:  # short row, extra field or non-integer: a parse error at that line (exit 4)
                raise TraceParseError(f"{path}: expected three integers 'layer,expert,device', got {row!r}",
                                      ln) from None
            if not (0 <= l < model.L and 0 <= e < model.E):
                raise ConfigError(f"{path}: ({l}, {e}) outside the model shape")
            assign[l, e] = s
    p = Placement(assign, c)
    if c is not None and n_devices is not None:
        v = validate(p, c, model, n_devices)
        if v:
            raise MoeplaceError(f"{path}: placement violates {len(v)} constraint(s), first: {v[0]}")
    return p
