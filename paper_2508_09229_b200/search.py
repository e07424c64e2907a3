"""GPU-driven placement search (extension beyond the reference).

Local search over placements: every iteration perturbs the incumbent into a batch of candidates
with random within-layer swaps (which keep every per-(device, layer) and per-device count, so
constraints stay satisfied — SPEC.md:182-191), scores the whole batch at once with the factorized
evaluator and accepts the best candidate if it improves the objective.  The whole iteration runs as
device kernels with no host synchronisation:

  * ``mp_perturb_pe_u8``   the candidates' per-expert cost rows: swapping two experts' devices swaps
                           their pe bytes, so a candidate is the incumbent's u8 row with its swaps
                           applied (the swap list is kept, the int32 assignments are never built);
  * ``mp_contract_tc_u8``  exact per-chunk hop sums of the batch on the tensor cores (tcgen05 kind::i8)
                           against the trace's per-chunk count digits, computed ONCE per search;
  * ``mp_batch_objective`` the objective of every candidate from its exact sums;
  * ``mp_search_accept``   argmin, and — if it improves — the winner's swaps replayed on the device
                           assignment and cost row; the history is written on the device.

Objectives are functions of the exact per-chunk hop sums, so they can be non-linear where the ILP
of Eq. (1) is linear:
  * "mean"       token-weighted mean hops (= K * objective_value; ILPLoad is optimal)
  * "mean+std"   mean + lam * population std of per-chunk means (robustness across dialogs)
  * "max"        worst per-chunk mean
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, MoeplaceError
from .eval import CountDigits, _pe_from_device_assign
from .model_trace import ActivationTrace, chunk_counts
from .placement import CostMatrix, Placement

OBJECTIVES = {"mean": 0, "mean+std": 1, "max": 2}


@dataclass
class SearchResult:
    placement: Placement
    objective: float
    history: list = field(default_factory=list)  # objective of the incumbent after each iteration
    evaluated: int = 0                          # candidates scored
    accepted: list = field(default_factory=list)  # per iteration: accepted candidate index or -1


def improve_placement(trace: ActivationTrace, start: Placement, cost: CostMatrix, objective: str = "mean",
                      lam: float = 1.0, iters: int = 50, batch: int = 1024, n_swaps: int = 2,
                      seed: int = 0) -> SearchResult:
    """Batched local search from `start` on `trace` (e.g. the train split)."""
    t = _lib.torch()
    m = trace.model
    if m is None or trace.n_tokens == 0:
        raise MoeplaceError("improve_placement: empty trace")
    if start.assign.shape != (m.L, m.E):
        raise ConfigError("placement shape does not match the trace")
    if objective not in OBJECTIVES:
        raise ConfigError(f"unknown objective {objective!r}")
    if batch < 1 or n_swaps < 1 or iters < 0:
        raise ConfigError("batch and n_swaps must be >= 1, iters >= 0")
    dev = _lib.require_cuda()
    C, LE = trace.n_chunks, m.L * m.E
    err = _lib.new_err()
    digits = CountDigits(chunk_counts(trace).view(C, -1), int(max(trace.chunk_token_counts().max(), 0)), err)
    tokens = _lib.to_dev(trace.chunk_token_counts(), t.int64)
    cur = _lib.to_dev(start.assign, t.int32)
    pe0 = _pe_from_device_assign(cur.unsqueeze(0), [cost], m)        # [1, LE] view of a padded row
    ldpe = -(-LE // 16) * 16
    pe_cur = t.zeros(ldpe, dtype=t.uint8, device=dev)
    pe_cur[:LE].copy_(pe0[0])
    pe_b = t.empty((batch, ldpe), dtype=t.uint8, device=dev)
    swaps = t.empty((batch, n_swaps, 3), dtype=t.int32, device=dev)
    sums = t.zeros((batch, C), dtype=t.int64, device=dev)
    obj = t.empty(batch, dtype=t.float64, device=dev)
    cur_obj = t.empty(1, dtype=t.float64, device=dev)
    history = t.empty(iters + 1, dtype=t.float64, device=dev)
    accepted = t.full((iters + 1,), -1, dtype=t.int64, device=dev)
    sh = _lib.stream_handle()
    kind = OBJECTIVES[objective]

    s0 = digits.contract(pe_cur.view(1, ldpe)[:, :LE], t.zeros((1, C), dtype=t.int64, device=dev))
    _lib.call("mp_batch_objective", _lib.ptr(s0), _lib.ptr(tokens), 1, C, kind, float(lam), _lib.ptr(cur_obj), sh)
    history[0:1].copy_(cur_obj)
    for it in range(iters):
        _lib.call("mp_perturb_pe_u8", _lib.ptr(pe_cur), m.L, m.E, batch, n_swaps, int(seed) & 0xFFFFFFFFFFFFFFFF, it,
                  _lib.ptr(pe_b), ldpe, _lib.ptr(swaps), sh)
        sums.zero_()
        digits.contract(pe_b[:, :LE], sums)
        _lib.call("mp_batch_objective", _lib.ptr(sums), _lib.ptr(tokens), batch, C, kind, float(lam), _lib.ptr(obj), sh)
        _lib.call("mp_search_accept", _lib.ptr(obj), batch, _lib.ptr(swaps), n_swaps, m.E, _lib.ptr(cur),
                  _lib.ptr(pe_cur), _lib.ptr(cur_obj), _lib.ptr(history), it + 1, _lib.ptr(accepted), sh)
    _lib.check_err(err, "improve_placement: per-chunk count outside its digit range")
    hist = history.cpu().tolist()
    out = Placement(cur.cpu().numpy(), start.constraints, (start.label or "start") + f"+search[{objective}]")
    return SearchResult(out, hist[-1], hist, 1 + iters * batch, accepted[1:].cpu().tolist())
