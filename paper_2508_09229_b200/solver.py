"""``moeplace.solver`` — ILP coefficients and the exact placement solver.

``build_instance`` builds the objective coefficients on the GPU (``mp_coeffs``: float64
w = f * p and the scaled integer costs rint(w * 1e9), bit-identical to numpy).
``solve_exact`` stays on the host (the ILP solve is not data parallel): a native min-cost flow
(``mp_solve_mcf``, csrc/solver.cpp) on the class-compressed FlowNetwork.
"""
from __future__ import annotations

import itertools
import json
import time
from dataclasses import dataclass, field
from typing import Any, Optional, Union

import numpy as np

from . import _lib
from .errors import ConfigError, InfeasibleError, MoeplaceError
from .model_trace import FrequencyTable
from .placement import Constraints, CostMatrix, Placement, validate

SCALE = 1e9  # cost integerisation


@dataclass
class PlacementInstance:
    """SPEC.md:259-262.  ``w`` float64 [L, E, S] and ``w_int`` = rint(w * scale) int64, both
    device tensors; ``p`` is the cost matrix the weights factor through (enables class
    compression in the flow network)."""

    w: Any
    w_int: Any
    constraints: Constraints
    L: int
    E: int
    S: int
    p: Optional[np.ndarray] = None
    scale: float = SCALE
    label: str = ""

    def w_numpy(self) -> np.ndarray:
        return self.w.cpu().numpy() if hasattr(self.w, "cpu") else np.asarray(self.w, dtype=np.float64)

    def w_int_numpy(self) -> np.ndarray:
        if self.w_int is None:
            return np.rint(self.w_numpy() * self.scale).astype(np.int64)
        return self.w_int.cpu().numpy() if hasattr(self.w_int, "cpu") else np.asarray(self.w_int, dtype=np.int64)


@dataclass
class FlowNetwork:
    """nodes source, items (l,e), slots (l,s), servers s, sink; arcs as
    (tail, head, capacity, cost).  Materialised for inspection/testing of small instances —
    the solver builds its own (compressed) network natively."""

    n_nodes: int
    arcs: list = field(default_factory=list)
    source: int = 0
    sink: int = 0


def flow_network(inst: PlacementInstance) -> FlowNetwork:
    L, E, S = inst.L, inst.E, inst.S
    w = inst.w_int_numpy()
    item0, slot0 = 1, 1 + L * E
    srv0 = slot0 + L * S
    sink = srv0 + S
    net = FlowNetwork(sink + 1, [], 0, sink)
    c = inst.constraints
    for i in range(L * E):
        net.arcs.append((0, item0 + i, 1, 0))
    for l in range(L):
        for e in range(E):
            for s in range(S):
                net.arcs.append((item0 + l * E + e, slot0 + l * S + s, 1, int(w[l, e, s])))
    for l in range(L):
        for s in range(S):
            net.arcs.append((slot0 + l * S + s, srv0 + s, c.c_layer, 0))
    for s in range(S):
        net.arcs.append((srv0 + s, sink, c.c_exp, 0))
    return net


Uniform = "uniform"


@dataclass(frozen=True)
class UniformFrequencies:
    """f[l, e] = 1/E for every expert: the load-agnostic ILP objective."""

    E: int


def build_instance(cost: CostMatrix, freq: Union[FrequencyTable, UniformFrequencies, str, None], c: Constraints,
                   E: Optional[int] = None, exact: bool = False) -> PlacementInstance:
    """w[l,e,s] = f[l,e] * p[l,s].  ``freq`` may be a FrequencyTable (ILPLoad),
    ``UniformFrequencies(E)`` or "uniform" with ``E=`` (ILP).  Computed on the GPU; when the
    table carries its integer counts the device derives f itself, bit-identical to numpy.
    ``exact=True`` makes the flow costs the exact integers count*p (p for uniform) instead of
    rint(w * 1e9): same optimal placements, no resolution loss beyond 1e7 tokens."""
    p = cost.p
    L, S = int(p.shape[0]), int(p.shape[1])
    scale = 0.0 if exact else SCALE
    if isinstance(freq, UniformFrequencies):
        return _instance(cost, None, 0, freq.E, c, None, "ilp", scale)
    if freq is None or (isinstance(freq, str) and freq == Uniform):
        if E is None:
            raise ConfigError("uniform build_instance needs the expert count E")
        return _instance(cost, None, 0, int(E), c, None, "ilp", scale)
    if not isinstance(freq, FrequencyTable):
        raise ConfigError("freq must be a FrequencyTable, UniformFrequencies or 'uniform'")
    f = np.asarray(freq.f, dtype=np.float64)
    if f.ndim != 2 or f.shape[0] != L:
        raise ConfigError(f"frequency table shape {f.shape} does not match cost matrix [{L}, {S}]")
    if (f < 0).any() or not np.isfinite(f).all():
        raise MoeplaceError("build_instance: negative or non-finite frequency")
    counts, denom = freq.counts, freq.topk * freq.n_tokens
    if counts is not None and denom > 0 and np.array_equal(np.asarray(counts) / denom, f):
        return _instance(cost, counts, denom, f.shape[1], c, None, "ilpload", scale)
    if exact:
        raise ConfigError("exact costs need a FrequencyTable that carries its integer counts")
    return _instance(cost, None, 0, f.shape[1], c, f, "ilpload")


def _instance(cost: CostMatrix, counts, denom: int, E: int, c: Constraints, f_float, label: str,
              scale: float = SCALE) -> PlacementInstance:
    t = _lib.torch()
    p = cost.p
    L, S = int(p.shape[0]), int(p.shape[1])
    dev = p.device
    w = t.empty((L, E, S), dtype=t.float64, device=dev)
    w_int = t.empty((L, E, S), dtype=t.int64, device=dev)
    if f_float is not None:
        # arbitrary float table: same formula, device multiply (no counts available)
        f = t.as_tensor(np.asarray(f_float, dtype=np.float64), device=dev)
        w.copy_(f[:, :, None] * p.to(t.float64)[:, None, :])
        w_int.copy_(t.round(w * SCALE).to(t.int64))
    else:
        cnt = None if counts is None else _lib.to_dev(counts, t.int64)
        _lib.call("mp_coeffs", _lib.ptr(cnt), int(denom), _lib.ptr(p), L, E, S, float(scale), _lib.ptr(w),
                  _lib.ptr(w_int), _lib.stream_handle())
    return PlacementInstance(w, w_int, c, L, E, S, p.cpu().numpy(), scale if scale > 0 else 1.0, label)


def solve_exact(inst: PlacementInstance) -> tuple[Placement, float]:
    """optimal placement by min-cost flow; objective = sum of w over the
    assignment (unscaled).  Infeasible instances raise ``InfeasibleError``."""
    L, E, S = inst.L, inst.E, inst.S
    c = inst.constraints
    if S * c.c_layer < E:
        raise InfeasibleError(f"c_layer: {S} devices x {c.c_layer} < E={E}")
    if S * c.c_exp < L * E:
        raise InfeasibleError(f"c_exp: {S} devices x {c.c_exp} < L*E={L * E}")
    w_int = np.ascontiguousarray(inst.w_int_numpy(), dtype=np.int64)
    p = None if inst.p is None else np.ascontiguousarray(inst.p, dtype=np.uint8)
    assign = np.empty((L, E), dtype=np.int32)
    obj = np.zeros(1, dtype=np.int64)
    flow = np.zeros(1, dtype=np.int64)
    t0 = time.perf_counter()
    st = _lib.call("mp_solve_mcf", _lib.host_ptr(w_int), None if p is None else _lib.host_ptr(p), L, E, S, c.c_layer,
                   c.c_exp, _lib.host_ptr(assign), _lib.host_ptr(obj), _lib.host_ptr(flow))
    inst_wall = time.perf_counter() - t0
    if st == _lib.MP_INFEASIBLE:
        raise InfeasibleError(f"max flow {int(flow[0])} < L*E = {L * E} (binding: c_exp/c_layer capacities)")
    placement = Placement(assign, c, inst.label or "exact")
    w = inst.w_numpy()
    objective = float(w[np.arange(L)[:, None], np.arange(E)[None, :], assign].sum())
    placement.solve_report = {"objective": objective, "wall_time_s": inst_wall, "flow_value": int(flow[0]),
                              "scaled": True, "objective_scaled": int(obj[0])}
    return placement, objective


def write_solve_report(placement: Placement, path) -> None:
    """JSON solve report {objective, wall_time_s, flow_value, scaled:true}."""
    rep = getattr(placement, "solve_report", None)
    if rep is None:
        raise ConfigError("placement has no solve report")
    with open(path, "w") as f:
        json.dump({k: rep[k] for k in ("objective", "wall_time_s", "flow_value", "scaled")}, f)


def brute_force_optimum(inst: PlacementInstance) -> float:
    """exhaustive minimum over all feasible assignments (guard S^(L*E) <= 1e7)."""
    L, E, S = inst.L, inst.E, inst.S
    if S ** (L * E) > 10 ** 7:
        raise ConfigError(f"brute force guard: S^(L*E) = {S}^{L * E} > 1e7")
    w = inst.w_numpy()
    c = inst.constraints
    best = None
    flat = w.reshape(L * E, S)
    layer_of = np.repeat(np.arange(L), E)
    for combo in itertools.product(range(S), repeat=L * E):
        a = np.asarray(combo)
        per_dev = np.bincount(a, minlength=S)
        if per_dev.max() > c.c_exp:
            continue
        per_layer = np.zeros((L, S), dtype=np.int64)
        np.add.at(per_layer, (layer_of, a), 1)
        if per_layer.max() > c.c_layer:
            continue
        v = float(flat[np.arange(L * E), a].sum())
        if best is None or v < best:
            best = v
    if best is None:
        raise InfeasibleError("no feasible assignment")
    return best
