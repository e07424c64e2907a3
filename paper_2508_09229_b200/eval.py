"""``moeplace.eval`` — the placement traffic evaluator.

``evaluate`` / ``evaluate_many`` score placements on the GPU: the placements' per-expert
round-trip hop costs pe_q[l, e] = p[l, assign_q[l, e]] are packed into u8 lanes
(``mp_pack_tables``) and ``mp_score_u8`` streams the trace once per group of up to 16
placements (32 where the count-contract kernel runs, see ``pass_lanes``), gathering pe_q for every (token, layer, pick) and reducing exact int64 hop sums per
chunk.  The host derives the report floats from those integers with numpy (the oracle runs the
same float code on its own integers, so reports are bit-identical, not merely within 1e-6).
"""
from __future__ import annotations

import json
import threading
from dataclasses import asdict, dataclass, field
from typing import Any, Optional, Sequence, Union

import numpy as np

from . import _lib
from .errors import ConfigError, MoeplaceError
from .model_trace import ActivationTrace, FrequencyTable, ModelSpec, chunk_counts, frequencies_from_counts, sweep
from .placement import CostMatrix, Placement

MAX_LANES = 16  # placements scored per pass by every algorithm (W = 4 words of four u8 lanes)
MAX_LANES_COUNT = 32  # per count-contract pass (W = 8): its per-placement work is per piece, not per byte
FACTORIZED_MAX_BYTES = 4 << 30  # evaluate_many(auto): largest per-chunk count array worth materialising


@dataclass
class EvalReport:
    """SPEC.md:326-329.  ``std_hops`` is the population std (ddof=0) of per-chunk means."""

    mean_hops_per_token: float
    std_hops: float
    n_tokens: int
    n_chunks: int
    objective_train: Optional[float] = None
    label: str = ""
    empty_chunks: int = 0
    hop_sum: int = 0                      # exact integer total (sum over tokens)
    chunk_hop_sums: Optional[list] = None  # exact per-chunk integers (id order)

    def to_json(self) -> dict:
        d = asdict(self)
        d.pop("chunk_hop_sums")
        return d

    def write(self, path) -> None:
        with open(path, "w") as f:
            json.dump(self.to_json(), f, indent=1, sort_keys=True)


@dataclass
class CommMap:
    """symmetric server x server hop volume per token, zero diagonal."""

    traffic: np.ndarray  # float64 [n_servers, n_servers]
    raw: Optional[np.ndarray] = None  # exact int64 directed accumulations (before /N and symmetrisation)

    def to_csv(self, path) -> None:
        n = self.traffic.shape[0]
        with open(path, "w") as f:
            f.write(",".join(str(i) for i in range(n)) + "\n")
            for r in range(n):
                f.write(",".join(repr(float(v)) for v in self.traffic[r]) + "\n")


def report_from_sums(sums: np.ndarray, tokens: np.ndarray, label: str = "") -> EvalReport:
    """EvalReport floats from exact integer per-chunk sums.  Empty chunks
    are excluded and counted."""
    sums = np.asarray(sums, dtype=np.int64)
    tokens = np.asarray(tokens, dtype=np.int64)
    keep = tokens > 0
    n_tok = int(tokens.sum())
    if n_tok == 0:
        raise MoeplaceError("evaluate: empty trace")
    total = int(sums.sum())
    means = sums[keep] / tokens[keep]
    return EvalReport(mean_hops_per_token=total / n_tok, std_hops=float(np.std(means)), n_tokens=n_tok,
                      n_chunks=int(keep.sum()), label=label, empty_chunks=int((~keep).sum()), hop_sum=total,
                      chunk_hop_sums=sums.tolist())


def _batch_floats(sums: np.ndarray, tokens: np.ndarray):
    """Row-wise EvalReport floats of int64 [P, C] per-chunk sums, bit-identical to
    ``report_from_sums`` per row: the per-chunk means form a C-contiguous [P, C'] array, so numpy's
    row reductions add in the same order as its 1-D ones, and totals / n_tokens is an exactly
    rounded division of exact integers (totals < 2^53 convert to float64 exactly; larger totals
    take Python's int division)."""
    sums = np.asarray(sums, dtype=np.int64)
    tokens = np.asarray(tokens, dtype=np.int64)
    keep = tokens > 0
    n_tok = int(tokens.sum())
    if n_tok == 0:
        raise MoeplaceError("evaluate: empty trace")
    totals = sums.sum(axis=1)
    if totals.size and int(np.abs(totals).max()) >= 2 ** 53:
        means = np.array([t / n_tok for t in totals.tolist()], dtype=np.float64)
    else:
        means = totals.astype(np.float64) / n_tok
    stds = np.std(np.ascontiguousarray(sums[:, keep]) / tokens[keep], axis=1)
    return totals, means, stds, n_tok, int(keep.sum()), int((~keep).sum())


def reports_from_sums(sums: np.ndarray, tokens: np.ndarray, labels: Sequence[str]) -> list[EvalReport]:
    """``report_from_sums`` for every row of int64 [P, C] at once (batched evaluation), same floats
    bit for bit (``_batch_floats``)."""
    sums = np.asarray(sums, dtype=np.int64)
    totals, means, stds, n_tok, n_chunks, n_empty = _batch_floats(sums, tokens)
    totals, means, stds = totals.tolist(), means.tolist(), stds.tolist()
    rows = sums.tolist()
    return [EvalReport(mean_hops_per_token=means[i], std_hops=stds[i], n_tokens=n_tok, n_chunks=n_chunks,
                       label=labels[i], empty_chunks=n_empty, hop_sum=totals[i], chunk_hop_sums=rows[i])
            for i in range(sums.shape[0])]


def _as_costs(costs, n: int) -> list[CostMatrix]:
    if isinstance(costs, CostMatrix):
        return [costs] * n
    costs = list(costs)
    if len(costs) != n:
        raise ConfigError(f"got {len(costs)} cost matrices for {n} placements")
    return costs


def _unique_costs(costs: Sequence[CostMatrix]):
    """Distinct cost matrices (by identity) and, per placement, the index of its matrix."""
    uniq: list[CostMatrix] = []
    topo_of = []
    for c in costs:
        for i, u in enumerate(uniq):
            if u is c:
                topo_of.append(i)
                break
        else:
            uniq.append(c)
            topo_of.append(len(uniq) - 1)
    return uniq, topo_of


def _stack_assign(placements: Sequence[Placement], costs: Sequence[CostMatrix], model: ModelSpec) -> np.ndarray:
    """int32 [P, L, E] assignments; shapes checked, and every expert placed on a device of its own
    placement's topology (cost matrices of different sizes can share one batch)."""
    out = np.empty((len(placements), model.L, model.E), dtype=np.int32)
    for i, (pl, c) in enumerate(zip(placements, costs)):
        a = np.asarray(pl.assign)
        if a.shape != (model.L, model.E):
            raise ConfigError(f"placement shape {a.shape} != model [{model.L}, {model.E}]")
        if a.size and (int(a.min()) < 0 or int(a.max()) >= c.S):
            raise MoeplaceError(f"evaluate: expert placed outside the topology (placement {i}, {c.S} devices)")
        out[i] = a
    return out


_STAGE = {"buf": None}            # pinned int32 staging for batched assignments (reused across calls)
_STAGE_LOCK = threading.Lock()
_STAGE_MAX_BYTES = 1 << 30          # larger batches use a one-off pinned buffer


def _assign_to_device(placements: Sequence[Placement], costs: Sequence[CostMatrix], model: ModelSpec):
    """Device int32 [P, L, E] assignments of a large batch, checked like ``_stack_assign`` (same
    errors): the host work is one memcpy per placement into a pinned staging buffer, and the
    per-placement range check runs on the device after one host-to-device copy."""
    t = _lib.torch()
    dev = _lib.require_cuda()
    P, L, E = len(placements), model.L, model.E
    nbytes = P * L * E * 4
    with _STAGE_LOCK:
        buf = _STAGE["buf"]
        if buf is None or buf.numel() < P * L * E:
            buf = t.empty(P * L * E, dtype=t.int32, pin_memory=True)
            if nbytes <= _STAGE_MAX_BYTES:
                _STAGE["buf"] = buf
        host = buf[:P * L * E].numpy().reshape(P, L, E)
        for i, pl in enumerate(placements):
            a = np.asarray(pl.assign)
            if a.shape != (L, E):
                raise ConfigError(f"placement shape {a.shape} != model [{L}, {E}]")
            if a.dtype != np.int32 and a.size and (int(a.min()) < 0 or int(a.max()) >= costs[i].S):
                raise MoeplaceError(f"evaluate: expert placed outside the topology (placement {i}, "
                                    f"{costs[i].S} devices)")  # checked before narrowing to int32
            np.copyto(host[i], a, casting="unsafe")
        out = buf[:P * L * E].to(dev, non_blocking=True).view(P, L, E)
        t.cuda.current_stream().synchronize()  # the staging buffer is free again
    return out


def _padded_costs(uniq: Sequence[CostMatrix], model: ModelSpec):
    """uint8 [T, L, S_max]: the distinct cost matrices, zero-padded to the widest topology."""
    t = _lib.torch()
    S = max(c.S for c in uniq)
    for c in uniq:
        if c.L != model.L:
            raise ConfigError(f"cost matrix has {c.L} layers, model has {model.L}")
    if all(c.S == S for c in uniq):
        return t.stack([c.p for c in uniq]).contiguous(), S
    cost = t.zeros((len(uniq), model.L, S), dtype=t.uint8, device=uniq[0].p.device)
    for i, c in enumerate(uniq):
        cost[i, :, :c.S] = c.p
    return cost, S


def _group_tables(placements: Sequence[Placement], costs: Sequence[CostMatrix], model: ModelSpec, W: int):
    """Pack one group (<= 4W placements) into device tables uint32 [L, 256, W]."""
    t = _lib.torch()
    dev = _lib.require_cuda()
    uniq, topo_of = _unique_costs(costs)
    cost, S = _padded_costs(uniq, model)
    assign = _stack_assign(placements, costs, model)
    d_assign = _lib.to_dev(assign, t.int32)
    d_topo = _lib.to_dev(np.asarray(topo_of, dtype=np.int32), t.int32)
    tables = t.empty((model.L, 256, W), dtype=t.int32, device=dev)
    err = _lib.new_err()
    _lib.call("mp_pack_tables", _lib.ptr(cost), len(uniq), _lib.ptr(d_assign), _lib.ptr(d_topo), len(placements),
              model.L, model.E, S, _lib.ptr(tables), W, _lib.ptr(err), _lib.stream_handle())
    _lib.check_err(err, "evaluate: unplaced expert")
    max_p = max(c.max_p for c in uniq)
    return tables, max_p


def _lanes_for(n: int) -> int:
    return 1 if n <= 4 else 2 if n <= 8 else 4 if n <= 16 else 8


def pass_lanes(trace: ActivationTrace, costs, algo: str = "auto", hist: bool = False) -> int:
    """Placements per scoring pass: 32 when the pass runs the count-contract kernel (``algo`` "count",
    or "auto" where the library picks it for this shape, i.e. long chunks) -- a 24-placement batch is
    then one pass, not two -- else 16."""
    if algo == "count":
        return MAX_LANES_COUNT
    if algo != "auto":
        return MAX_LANES
    m = trace.model
    if m is None or trace.n_tokens == 0:
        return MAX_LANES
    cs = [costs] if isinstance(costs, CostMatrix) else list(costs)
    max_p = max((c.max_p for c in _unique_costs(cs)[0]), default=0)
    auto = _lib.choose_algo(hist, 4, trace.n_tokens, trace.n_chunks, m.L, m.K, max_p)
    return MAX_LANES_COUNT if auto == "count" else MAX_LANES


ALGOS = {"auto": 0, "gather": 1, "count": 2, "token": 3, "seg": 4}  # include/moeplace_cuda.h MP_ALGO_*


def score_sums(trace: ActivationTrace, placements: Sequence[Placement], costs, algo: str = "auto") -> np.ndarray:
    """Exact per-chunk hop sums, int64 [P, C], computed on the GPU (``mp_score_ex_u8``), up to 16
    placements per pass (32 per count-contract pass, ``pass_lanes``).  ``algo``: "gather" (per-byte table lookups), "count" (count-contract:
    per-(layer, chunk) histograms contracted with the tables), "token" (token-tiled: per-token sums
    across layers reduced per chunk; cost independent of the chunk count), "seg" (segmented gather:
    warps own contiguous token ranges and reduce at each chunk boundary; C-independent, K = 8 and
    costs <= 31) or "auto" (the library's choice for the shape); all give the same integers."""
    if algo not in ALGOS:
        raise ConfigError(f"unknown score algorithm {algo!r}")
    t = _lib.torch()
    m = trace.model
    if m is None or trace.n_tokens == 0:
        raise MoeplaceError("evaluate: empty trace")
    placements = list(placements)
    costs = _as_costs(costs, len(placements))
    C = trace.n_chunks
    dev = _lib.require_cuda()
    groups = []
    lanes = pass_lanes(trace, costs, algo)
    for g0 in range(0, len(placements), lanes):
        grp = placements[g0:g0 + lanes]
        W = _lanes_for(len(grp))
        tables, max_p = _group_tables(grp, costs[g0:g0 + lanes], m, W)
        groups.append((g0, len(grp), W, tables, max_p, t.zeros((4 * W, C), dtype=t.int64, device=dev)))

    def launch(planes, stride, t0, t1, bounds):
        for _, _, W, tables, max_p, sums in groups:
            _lib.call("mp_score_ex_u8", _lib.ptr(planes), stride, t0, t1, m.L, m.K, _lib.ptr(bounds), C,
                      _lib.ptr(tables), W, max_p, _lib.ptr(sums), ALGOS[algo], _lib.stream_handle())

    sweep(trace, launch)
    out = np.zeros((len(placements), C), dtype=np.int64)
    for g0, n, _, _, _, sums in groups:
        out[g0:g0 + n] = sums[:n].cpu().numpy()
    return out


def pe_matrix(placements: Sequence[Placement], costs, model: ModelSpec):
    """uint8 [P, L*E] per-expert round-trip costs pe_q[l, e] = p_q[l, assign_q[l, e]] on the device
    (``mp_pe_gather_u8``; rows padded to a 16-byte pitch, the returned tensor is the [P, L*E] view)."""
    placements = list(placements)
    costs = _as_costs(costs, len(placements))
    return _pe_from_device_assign(_assign_to_device(placements, costs, model), costs, model)


def _pe_from_device_assign(assign, costs: Sequence[CostMatrix], model: ModelSpec):
    """pe uint8 [P, L*E] (a view of a [P, ldpe] buffer, ldpe = L*E rounded up to 16) from device
    assignments [P, L, E] (``mp_pe_gather_u8``, one launch for every topology of the batch); an
    expert placed outside its placement's topology raises the SPEC error."""
    t = _lib.torch()
    dev = _lib.require_cuda()
    uniq, topo_of = _unique_costs(costs)
    cost, S = _padded_costs(uniq, model)
    P, LE = assign.shape[0], model.L * model.E
    ldpe = -(-LE // 16) * 16
    a32 = assign.to(device=dev, dtype=t.int32).contiguous()
    d_topo = _lib.to_dev(np.asarray(topo_of, dtype=np.int32), t.int32)
    d_S = _lib.to_dev(np.asarray([c.S for c in uniq], dtype=np.int32), t.int32)
    pe = t.empty((P, ldpe), dtype=t.uint8, device=dev)
    err = _lib.new_err()
    _lib.call("mp_pe_gather_u8", _lib.ptr(cost), len(uniq), model.L, S, _lib.ptr(d_S), _lib.ptr(a32), _lib.ptr(d_topo),
              P, model.E, _lib.ptr(pe), ldpe, _lib.ptr(err), _lib.stream_handle())
    code, q, _, _ = _lib.read_err(err)
    if code:
        raise MoeplaceError(f"evaluate: expert placed outside the topology (placement {q}, {costs[q].S} devices)")
    return pe[:, :LE]


def _pe_operand(pe):
    """(tensor, row pitch) of a uint8 [P, LE] cost matrix as the contraction's A operand: rows with a
    16-byte-multiple pitch (a padded copy only when the given rows do not have one)."""
    t = _lib.torch()
    P, LE = pe.shape
    if pe.stride(1) == 1 and pe.stride(0) % 16 == 0 and pe.data_ptr() % 16 == 0:
        return pe, pe.stride(0)
    ldpe = -(-LE // 16) * 16
    A = t.zeros((P, ldpe), dtype=t.uint8, device=pe.device)
    A[:, :LE].copy_(pe)
    return A, ldpe


def _n_digits(max_count: int) -> int:
    if max_count < 0:
        raise ConfigError("contract_tc: negative count bound")
    for nd in (1, 2, 4):
        if max_count < (1 << (8 * nd)):
            return nd
    raise ConfigError("contract_tc: per-chunk counts of 2^32 or more are outside the digit format")


class CountDigits:
    """The contraction's B operand: per-chunk counts int64 [C, LE] split into 8-bit digits
    (``mp_count_digits_u8``), uint8 [C*ndig, ldd], row c*ndig + a = digit a of chunk c.  Built once
    per trace (the placement search reuses it every iteration)."""

    def __init__(self, cnt, max_count: Optional[int] = None, err=None):
        t = _lib.torch()
        C, LE = cnt.shape
        if max_count is None:
            max_count = int(cnt.max().item()) if cnt.numel() else 0
        self.C, self.LE, self.ndig = C, LE, _n_digits(int(max_count))
        self.ldd = -(-LE // 16) * 16
        self.buf = t.empty((C * self.ndig, self.ldd), dtype=t.uint8, device=cnt.device)
        self.err = _lib.new_err() if err is None else err
        self.own_err = err is None
        _lib.call("mp_count_digits_u8", _lib.ptr(cnt.contiguous()), C, LE, self.ndig, self.ldd, _lib.ptr(self.buf),
                  _lib.ptr(self.err), _lib.stream_handle())

    def contract(self, pe, out=None, ctas: int = 0):
        """out[P, C] += pe [P, LE] @ counts^T, exact int64, on the tensor cores (``mp_contract_tc_u8``;
        ``ctas`` = 0: one CTA per SM)."""
        t = _lib.torch()
        A, ldpe = _pe_operand(pe)
        P = A.shape[0]
        if out is None:
            out = t.zeros((P, self.C), dtype=t.int64, device=A.device)
        _lib.call("mp_contract_tc_u8", _lib.ptr_any(A), P, ldpe, _lib.ptr(self.buf), self.C, self.ndig, self.LE,
                  self.ldd, _lib.ptr(out), ctas, _lib.stream_handle())
        return out

    def check(self):
        if self.own_err:
            _lib.check_err(self.err, "contract_tc: per-chunk count outside its digit range")


def contract_tc(cnt, pe, max_count: Optional[int] = None, max_pe: Optional[int] = None, err=None):
    """Exact hop sums [P, C] = pe [P, LE] (uint8) @ cnt^T [LE, C] (int64 per-chunk counts) on the 5th-
    generation tensor cores: the counts are split into 8-bit digits (``mp_count_digits_u8``) and ONE
    u8 x u8 GEMM (``mp_contract_tc_u8``: tcgen05 kind::i8, TMA-fed, int32 accumulators in TMEM, exact
    split-K ranges) produces every digit's partials, recombined into int64 in its epilogue.
    ``max_count`` bounds the counts (no device reduction or sync when given; a count above it raises
    rather than truncating); ``max_pe`` is accepted for compatibility (pe is used as u8 as it is);
    with ``err`` the caller checks that device error block itself."""
    d = CountDigits(cnt, max_count, err)
    out = d.contract(pe)
    d.check()
    return out


def score_sums_factorized(trace: ActivationTrace, placements: Sequence[Placement], costs,
                          contraction: str = "tc") -> np.ndarray:
    """Per-chunk hop sums via the factorized evaluator: one per-chunk histogram pass
    (``mp_hist_chunks_u8``) and an exact integer contraction with every placement's per-expert
    costs — on the tensor cores (``contraction="tc"``: 7-bit-digit int8 GEMMs, cuBLASLt) or with
    the CUDA-core int64 kernel ``mp_contract_counts`` (``"cuda"``).  Bit-identical to
    ``score_sums`` by linearity; cost independent of P per token.  A cross-check
    and the fast path for large candidate batches — it produces no per-token values (use
    ``token_hops_all`` / ``evaluate_dedup`` for those)."""
    t = _lib.torch()
    m = trace.model
    if m is None or trace.n_tokens == 0:
        raise MoeplaceError("evaluate: empty trace")
    cnt = chunk_counts(trace)
    C = trace.n_chunks
    pe = pe_matrix(placements, costs, m)
    if contraction == "tc":
        # a per-chunk count is at most the chunk's token count (distinct picks per record)
        max_count = int(np.max(trace.chunk_token_counts()))
        out = contract_tc(cnt.view(C, -1), pe, max_count=max_count)
    elif contraction == "cuda":
        out = t.zeros((pe.shape[0], C), dtype=t.int64, device=cnt.device)
        pe_c = pe.contiguous()
        _lib.call("mp_contract_counts", _lib.ptr(cnt), C, _lib.ptr(pe_c), pe.shape[0], m.L * m.E, _lib.ptr(out),
                  _lib.stream_handle())
    else:
        raise ConfigError(f"unknown contraction {contraction!r}")
    return out.cpu().numpy()


def evaluate_many(trace: ActivationTrace, placements: Sequence[Placement], costs,
                  method: str = "auto") -> list[EvalReport]:
    """Batched ``evaluate`` over placements (and per-placement cost matrices, i.e. topologies),
    extension A18.  ``method``: "gather" / "count" / "token" — passes of up to 16 (count: 32) placements with
    that algorithm; "factorized" — one per-chunk histogram pass + tensor-core contraction for any
    number of placements; "auto" — passes (the library picks the algorithm per pass) when P fits one
    pass (``pass_lanes``: 32 on long chunks, 16 on short ones) or the per-chunk counts would exceed
    FACTORIZED_MAX_BYTES, factorized otherwise.  All give
    identical integers."""
    placements = list(placements)
    if method == "auto":
        # factorized materialises int64 [C, L, E] per-chunk counts: worth it for large batches, but
        # not when short chunks make that array huge (then the library's own choice per pass --
        # token-tiled for short chunks -- is the better way)
        m = trace.model
        fact_bytes = trace.n_chunks * (m.L * m.E if m else 0) * 8
        lanes = pass_lanes(trace, _as_costs(costs, len(placements)))
        method = "factorized" if len(placements) > lanes and fact_bytes <= FACTORIZED_MAX_BYTES else "pass"
    if method in ("gather", "count", "token", "pass"):
        sums = score_sums(trace, placements, costs, algo="auto" if method == "pass" else method)
    elif method == "factorized":
        sums = score_sums_factorized(trace, placements, costs)
    else:
        raise ConfigError(f"unknown evaluate method {method!r}")
    return reports_from_sums(sums, trace.chunk_token_counts(), [p.label for p in placements])


@dataclass
class BatchReport:
    """``evaluate_batch`` result: the EvalReport fields of P placements as arrays, row q = placement
    q (same values, bit for bit, as ``evaluate_many``'s EvalReports)."""

    mean_hops_per_token: np.ndarray  # float64 [P]
    std_hops: np.ndarray             # float64 [P]
    hop_sum: np.ndarray              # int64 [P], exact
    chunk_hop_sums: np.ndarray       # int64 [P, C], exact, chunk id order
    n_tokens: int
    n_chunks: int
    empty_chunks: int

    def report(self, q: int, label: str = "") -> EvalReport:
        return EvalReport(mean_hops_per_token=float(self.mean_hops_per_token[q]), std_hops=float(self.std_hops[q]),
                          n_tokens=self.n_tokens, n_chunks=self.n_chunks, label=label,
                          empty_chunks=self.empty_chunks, hop_sum=int(self.hop_sum[q]),
                          chunk_hop_sums=self.chunk_hop_sums[q].tolist())


def evaluate_batch(trace: ActivationTrace, assign, costs, method: str = "auto") -> BatchReport:
    """``evaluate_many`` for a candidate batch given as one integer array ``assign`` [P, L, E]
    (numpy or torch, host or device; e.g. ``placement.perturb_swaps`` output), extension A18 for
    search loops: the batch moves to the device in one copy, is range-checked there, and the
    result is arrays instead of P report objects.  ``costs``: one CostMatrix, or one per
    placement.  ``method`` as in ``evaluate_many``."""
    t = _lib.torch()
    m = trace.model
    if m is None or trace.n_tokens == 0:
        raise MoeplaceError("evaluate: empty trace")
    dev = _lib.require_cuda()
    a = assign if isinstance(assign, t.Tensor) else t.from_numpy(np.ascontiguousarray(assign))
    if a.dim() != 3 or tuple(a.shape[1:]) != (m.L, m.E):
        raise ConfigError(f"assign batch shape {tuple(a.shape)} != [P, {m.L}, {m.E}]")
    if a.dtype.is_floating_point or a.dtype == t.bool:
        raise ConfigError("assign batch must hold integer device ids")
    P = int(a.shape[0])
    costs = _as_costs(costs, P)
    if a.dtype != t.int32 and a.numel():  # range-check before narrowing to int32 (the gather checks the rest)
        lo, hi = int(a.min()), int(a.max())
        if lo < 0 or hi >= 2 ** 31:
            raise MoeplaceError("evaluate: expert placed outside the topology")
    a = a.to(dev, non_blocking=a.is_pinned())
    if method == "auto":
        fact_bytes = trace.n_chunks * m.L * m.E * 8
        method = "factorized" if P > pass_lanes(trace, costs) and fact_bytes <= FACTORIZED_MAX_BYTES else "pass"
    if method == "factorized":
        pe = _pe_from_device_assign(a, costs, m)  # checks every assignment against its topology
        cnt = chunk_counts(trace)
        sums = contract_tc(cnt.view(trace.n_chunks, -1), pe,
                           max_count=int(np.max(trace.chunk_token_counts()))).cpu().numpy()
    elif method in ("gather", "count", "token", "pass"):
        _pe_from_device_assign(a, costs, m)  # same range check as the factorized path
        host = a.to(t.int32).cpu().numpy()
        pls = [Placement(host[q]) for q in range(P)]
        sums = score_sums(trace, pls, costs, algo="auto" if method == "pass" else method)
    else:
        raise ConfigError(f"unknown evaluate method {method!r}")
    totals, means, stds, n_tok, n_chunks, n_empty = _batch_floats(sums, trace.chunk_token_counts())
    return BatchReport(means, stds, totals, np.asarray(sums, dtype=np.int64), n_tok, n_chunks, n_empty)


def evaluate(trace: ActivationTrace, placement: Placement, cost: CostMatrix) -> EvalReport:
    """per-chunk hop sums on the GPU; mean = token-weighted grand mean, std =
    std of per-chunk means; empty chunks excluded with a warning count."""
    return evaluate_many(trace, [placement], cost)[0]


def evaluate_with_stats(trace: ActivationTrace, placements: Sequence[Placement], cost, algo: str = "auto"):
    """One fused pass (``mp_hist_score_ex_u8``): the trace's FrequencyTable plus the EvalReports of
    up to 16 placements, 32 where the pass runs count-contract (``pass_lanes``; ``cost``: one
    CostMatrix or one per placement).  Used for the train
    split, where the ILPLoad frequencies and the train-side metric come from the same tokens.
    ``algo`` as in ``score_sums`` ("gather" takes at most 4 placements)."""
    t = _lib.torch()
    m = trace.model
    placements = list(placements)
    if m is None or trace.n_tokens == 0:
        raise MoeplaceError("evaluate: empty trace")
    if algo not in ALGOS:
        raise ConfigError(f"unknown score algorithm {algo!r}")
    top = 4 if algo == "gather" else pass_lanes(trace, _as_costs(cost, len(placements)), algo, hist=True)
    if not 1 <= len(placements) <= top:
        raise ConfigError(f"evaluate_with_stats takes 1..{top} placements here")
    dev = _lib.require_cuda()
    W = _lanes_for(len(placements))
    tables, max_p = _group_tables(placements, _as_costs(cost, len(placements)), m, W)
    C = trace.n_chunks
    counts = t.zeros((m.L, m.E), dtype=t.int64, device=dev)
    sums = t.zeros((4 * W, C), dtype=t.int64, device=dev)
    err = _lib.new_err()

    def launch(planes, stride, t0, t1, bounds):
        _lib.call("mp_hist_score_ex_u8", _lib.ptr(planes), stride, t0, t1, m.L, m.K, m.E, _lib.ptr(bounds), C,
                  _lib.ptr(tables), W, max_p, _lib.ptr(counts), _lib.ptr(sums), _lib.ptr(err), ALGOS[algo],
                  _lib.stream_handle())

    sweep(trace, launch)
    _lib.check_err(err, "evaluate_with_stats")
    freq = frequencies_from_counts(counts.cpu().numpy(), trace.n_tokens, m.K)
    s = sums.cpu().numpy()
    tokens = trace.chunk_token_counts()
    return freq, [report_from_sums(s[i], tokens, placements[i].label) for i in range(len(placements))]


@dataclass
class DedupReport:
    """Extension A17 (north_star): per-token unique destination servers and deduplicated hops
    (one message per destination server).  ``spec`` is the unchanged SPEC EvalReport — the
    deduplicated numbers never replace it (SPEC.md:339 counts every selected expert)."""

    spec: EvalReport
    unique_dest_per_token: float
    dedup_hops_per_token: float
    label: str = ""
    chunk_uniq_sums: Optional[list] = None
    chunk_dedup_sums: Optional[list] = None


def evaluate_dedup(trace: ActivationTrace, placements: Sequence[Placement], costs) -> list[DedupReport]:
    """SPEC hops plus unique-destination counts per (token, layer) for each placement, in one
    pass per group of 4 placements (``mp_score_dedup_u8``).  Each cost matrix must carry its
    DistanceMatrix and AttentionPlacement (the server map and the dispatch servers)."""
    t = _lib.torch()
    m = trace.model
    if m is None or trace.n_tokens == 0:
        raise MoeplaceError("evaluate_dedup: empty trace")
    placements = list(placements)
    costs = _as_costs(costs, len(placements))
    dev = _lib.require_cuda()
    C = trace.n_chunks
    tokens = trace.chunk_token_counts()
    out = []
    for g0 in range(0, len(placements), 4):
        grp, gcost = placements[g0:g0 + 4], costs[g0:g0 + 4]
        for c in gcost:
            if c.dist is None or c.attn is None:
                raise ConfigError("evaluate_dedup needs cost matrices built by cost_matrix(dist, attn)")
            if c.dist.graph.n_servers > 256:  # server ids are one byte in the dedup tables
                raise ConfigError(f"evaluate_dedup supports at most 256 servers, topology has "
                                  f"{c.dist.graph.n_servers}")
        tables, max_p = _group_tables(grp, gcost, m, 1)
        uniq, topo_of = _unique_costs(gcost)
        S = max(c.S for c in uniq)
        srv = np.zeros((len(uniq), S), dtype=np.int32)  # zero-padded to the widest topology
        for i, c in enumerate(uniq):
            srv[i, :c.S] = c.dist.graph.device_server
        server_of = _lib.to_dev(srv, t.int32)
        d_assign = _lib.to_dev(_stack_assign(grp, gcost, m), t.int32)
        d_topo = _lib.to_dev(np.asarray(topo_of, dtype=np.int32), t.int32)
        srv_tables = t.empty((m.L, 256), dtype=t.int32, device=dev)
        err = _lib.new_err()
        _lib.call("mp_pack_server_tables", _lib.ptr(server_of), len(uniq), _lib.ptr(d_assign), _lib.ptr(d_topo),
                  len(grp), m.L, m.E, S, _lib.ptr(srv_tables), _lib.ptr(err), _lib.stream_handle())
        _lib.check_err(err, "evaluate_dedup: unplaced expert")
        src = np.zeros((4, m.L), dtype=np.uint8)
        for q, c in enumerate(gcost):
            src[q] = c.dist.graph.device_server[c.attn.dispatch]
        d_src = _lib.to_dev(src, t.uint8)
        hop = t.zeros((4, C), dtype=t.int64, device=dev)
        uq = t.zeros((4, C), dtype=t.int64, device=dev)
        dd = t.zeros((4, C), dtype=t.int64, device=dev)

        def launch(planes, stride, t0, t1, bounds):
            _lib.call("mp_score_dedup_u8", _lib.ptr(planes), stride, t0, t1, m.L, m.K, _lib.ptr(bounds), C,
                      _lib.ptr(tables), _lib.ptr(srv_tables), _lib.ptr(d_src), _lib.ptr(hop), _lib.ptr(uq),
                      _lib.ptr(dd), _lib.stream_handle())

        sweep(trace, launch)
        h, u, d = hop.cpu().numpy(), uq.cpu().numpy(), dd.cpu().numpy()
        for i, pl in enumerate(grp):
            out.append(DedupReport(report_from_sums(h[i], tokens, pl.label), int(u[i].sum()) / trace.n_tokens,
                                   int(d[i].sum()) / trace.n_tokens, pl.label, u[i].tolist(), d[i].tolist()))
    return out


def token_hops_all(trace: ActivationTrace, placements: Sequence[Placement], costs) -> np.ndarray:
    """``token_hops`` of EVERY token of the trace for each placement:
    int64 [P, N], from the token-tiled device kernel ``mp_token_hops_u8`` (4 placements per pass).
    Per-token values are what per-chunk sums cannot give: hop distributions, percentiles, tails."""
    t = _lib.torch()
    m = trace.model
    if m is None or trace.n_tokens == 0:
        raise MoeplaceError("token_hops_all: empty trace")
    placements = list(placements)
    costs = _as_costs(costs, len(placements))
    n = trace.n_tokens
    dev = _lib.require_cuda()
    out = np.zeros((len(placements), n), dtype=np.int64)
    for g0 in range(0, len(placements), 4):
        grp = placements[g0:g0 + 4]
        tables, max_p = _group_tables(grp, costs[g0:g0 + 4], m, 1)
        scratch = t.empty((m.L, 256, 32), dtype=t.int32, device=dev)
        done = [0]

        def launch(planes, stride, t0, t1, bounds):  # per-token outputs land at the slice's offset
            hops = t.empty((4, t1 - t0), dtype=t.int32, device=dev)
            _lib.call("mp_token_hops_u8", _lib.ptr(planes), stride, t0, t1, m.L, m.K, _lib.ptr(tables), max_p,
                      _lib.ptr(scratch), _lib.ptr(hops), _lib.stream_handle())
            o = done[0]
            out[g0:g0 + len(grp), o:o + t1 - t0] = hops[:len(grp)].cpu().numpy()
            done[0] = o + t1 - t0

        sweep(trace, launch)
    return out


def hop_distribution(trace: ActivationTrace, placement: Placement, cost: CostMatrix) -> np.ndarray:
    """Histogram of per-token hops: out[h] = number of tokens whose token_hops == h."""
    h = token_hops_all(trace, [placement], cost)[0]
    return np.bincount(h)


def token_hops(selections, placement: Placement, cost: CostMatrix) -> int:
    """sum over layers and selected experts of p[l, device(l, e)] for ONE token
    (``selections`` = L lists of selected experts).  Runs through the device scorer."""
    sel = [list(s) for s in selections]
    L, E = placement.assign.shape
    if len(sel) != L or not sel:
        raise ConfigError(f"selections must list {L} layers")
    K = len(sel[0])
    if any(len(s) != K for s in sel):
        raise ConfigError("every layer must select the same number of experts")
    arr = np.asarray(sel, dtype=np.int64).reshape(1, L, K)
    if arr.min() < 0 or arr.max() >= E:
        raise MoeplaceError("token_hops: expert index is not placed (outside [0, E))")
    tr = ActivationTrace.from_tokens(ModelSpec(L, E, K), arr.astype(np.uint8))
    return int(score_sums(tr, [placement], cost)[0].sum())


def objective_value(placement: Placement, freq: FrequencyTable, cost: CostMatrix) -> float:
    """sum_{l,e} f[l,e] * p[l, device(l,e)].  Equals evaluate(train).mean / K
    for the trace f was estimated from.  On the device: pe by ``mp_pe_gather_u8``;
    with the table's exact counts the sum is the integer contraction sum_{l,e} count * pe
    (``mp_contract_counts``) over K * n_tokens, one correctly rounded division; float-only
    frequencies are summed by ``mp_objective_f64``."""
    t = _lib.torch()
    f = np.asarray(freq.f, dtype=np.float64)
    a = np.asarray(placement.assign)
    if f.shape != a.shape:
        raise ConfigError(f"frequency table {f.shape} and placement {a.shape} differ")
    if a.size and (a.min() < 0 or a.max() >= cost.S):
        raise MoeplaceError("objective_value: expert placed outside the topology")
    L, E = a.shape
    model = ModelSpec(L, E, max(1, int(freq.topk or 1)))
    pe = _pe_from_device_assign(_lib.to_dev(a[None], t.int32), [cost], model)
    LE = L * E
    sh = _lib.stream_handle()
    if freq.counts is not None and freq.n_tokens and freq.topk:
        cnt = _lib.to_dev(np.asarray(freq.counts, dtype=np.int64).reshape(1, LE), t.int64)
        out = t.zeros((1, 1), dtype=t.int64, device=cnt.device)
        pe_c = pe.contiguous()
        _lib.call("mp_contract_counts", _lib.ptr(cnt), 1, _lib.ptr(pe_c), 1, LE, _lib.ptr(out), sh)
        return int(out.item()) / (int(freq.topk) * int(freq.n_tokens))
    fd = _lib.to_dev(f.reshape(LE), t.float64)
    out = t.empty(1, dtype=t.float64, device=fd.device)
    A, ldpe = _pe_operand(pe)
    _lib.call("mp_objective_f64", _lib.ptr(fd), _lib.ptr_any(A), ldpe, LE, 1, _lib.ptr(out), sh)
    return float(out.item())


def gain(baseline_hops: float, method_hops: float) -> float:
    """100 * (baseline - method) / method, in percent."""
    if not method_hops > 0:
        raise ConfigError(f"gain: method_hops must be positive, got {method_hops}")
    return 100.0 * (baseline_hops - method_hops) / method_hops


def communication_map(trace: ActivationTrace, placement: Placement, topology: Union[CostMatrix, tuple]) -> CommMap:
    """SPEC.md:371-379.  ``topology`` is the CostMatrix (it carries the distance matrix and the
    attention placement) or a (DistanceMatrix, AttentionPlacement) pair.  Accumulated on the GPU
    from the trace's exact (l, e) load counts (the map is linear in them)."""
    from .model_trace import trace_counts
    t = _lib.torch()
    if isinstance(topology, CostMatrix):
        dist, attn = topology.dist, topology.attn
    else:
        dist, attn = topology
    if dist is None or attn is None:
        raise ConfigError("communication_map needs the distance matrix and the attention placement")
    m = trace.model
    if m is None or trace.n_tokens == 0:
        raise MoeplaceError("communication_map: empty trace")
    g = dist.graph
    counts = trace_counts(trace)
    n = g.n_servers
    traffic = t.zeros((n, n), dtype=t.int64, device=counts.device)
    # keep every argument tensor referenced until the launch is enqueued (the caching allocator
    # would otherwise hand a freed temporary's memory to the next argument)
    d_assign = _lib.to_dev(placement.assign, t.int32)
    d_server = _lib.to_dev(g.device_server, t.int32)
    d_disp = _lib.to_dev(attn.dispatch, t.int32)
    d_coll = _lib.to_dev(attn.collect, t.int32)
    err = _lib.new_err()
    _lib.call("mp_comm_map", _lib.ptr(counts), _lib.ptr(d_assign), _lib.ptr(d_server), _lib.ptr(dist.server_dist), n,
              _lib.ptr(d_disp), _lib.ptr(d_coll), m.L, m.E, g.n_devices, _lib.ptr(traffic), _lib.ptr(err),
              _lib.stream_handle())
    _lib.check_err(err, "communication_map")
    raw = traffic.cpu().numpy()
    sym = (raw + raw.T) / 2.0 / trace.n_tokens
    return CommMap(sym, raw)
