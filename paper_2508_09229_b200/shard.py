"""Token-sharded multi-GPU evaluation.

The token dimension shards naturally: rank r owns tokens [r*N/G, (r+1)*N/G) of the trace (a
contiguous range that may cut through chunks), generates them in place (the generator is
counter-based, so a shard is bit-identical to the same tokens of the full trace), runs the fused
statistics+scoring pass, and the per-rank integer partials — the [L, E] load counts and the
[P, C] per-chunk hop sums, packed into ONE int64 buffer — are summed with a single
``torch.distributed.all_reduce`` (NCCL over NVLink on GPUs; gloo works for host tensors).
Integer sums are exact for any world size and any partition, so every rank ends with the same
bits as a single-GPU run; the report floats are then derived once, identically everywhere.
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .errors import ConfigError


def shard_range(n_tokens: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous token range of ``rank``: [floor(r*N/G), floor((r+1)*N/G))."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} for world size {world}")
    return (rank * n_tokens) // world, ((rank + 1) * n_tokens) // world


class Packed:
    """One int64 buffer holding [counts (L*E) | hop sums (P*C)]: a single collective per pass."""

    def __init__(self, L: int, E: int, P: int, C: int, device=None):
        import torch
        self.L, self.E, self.P, self.C = L, E, P, C
        self.buf = torch.zeros(L * E + P * C, dtype=torch.int64, device=device)

    @property
    def counts(self):
        return self.buf[: self.L * self.E].view(self.L, self.E)

    @property
    def sums(self):
        return self.buf[self.L * self.E:].view(self.P, self.C)

    def allreduce(self, group=None) -> "Packed":
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=group)
        return self


def sharded_evaluate(model, zipf_s: float, n_tokens: int, n_chunks: int, seed: int,
                     placements: Sequence, costs, group=None, rank: Optional[int] = None,
                     world: Optional[int] = None):
    """Generate this rank's shard on its GPU, build the load counts and the per-chunk hop sums of
    every placement (``costs``: one CostMatrix or one per placement — several topologies can be
    mixed), all-reduce ONE packed int64 buffer, and return the global
    (FrequencyTable, [EvalReport]) — identical on every rank and to a one-GPU run.
    Placements 0..15 ride the fused statistics pass; further ones are scored 16 per pass."""
    import torch
    import torch.distributed as dist

    from . import _lib
    from .eval import MAX_LANES, _as_costs, _group_tables, _lanes_for, report_from_sums
    from .model_trace import chunk_bounds_even, frequencies_from_counts, generate_trace

    if rank is None or world is None:
        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        else:
            rank, world = 0, 1
    placements = list(placements)
    if not placements:
        raise ConfigError("sharded_evaluate needs at least one placement")
    costs = _as_costs(costs, len(placements))
    a, b = shard_range(n_tokens, rank, world)
    tr = generate_trace(model, zipf_s, n_tokens, n_chunks, seed, tok_range=(a, b))
    dev = tr.planes.device
    P = len(placements)
    pk = Packed(model.L, model.E, P, n_chunks, dev)
    if b > a:
        planes, stride = tr.planes, tr.planes.shape[1]
        bounds = _lib.to_dev(tr.chunk_bounds, torch.int64)
        err = _lib.new_err()
        sh = _lib.stream_handle()
        head = placements[:MAX_LANES]
        W = _lanes_for(len(head))
        tables, max_p = _group_tables(head, costs[:MAX_LANES], model, W)
        sums = torch.zeros((4 * W, n_chunks), dtype=torch.int64, device=dev)
        _lib.call("mp_hist_score_ex_u8", _lib.ptr(planes), stride, 0, b - a, model.L, model.K, model.E,
                  _lib.ptr(bounds), n_chunks, _lib.ptr(tables), W, max_p, _lib.ptr(pk.counts), _lib.ptr(sums),
                  _lib.ptr(err), 0, sh)
        _lib.check_err(err, "sharded_evaluate")
        pk.sums[:len(head)].copy_(sums[:len(head)])
        for g0 in range(MAX_LANES, P, MAX_LANES):
            grp = placements[g0:g0 + MAX_LANES]
            W = _lanes_for(len(grp))
            tables, max_p = _group_tables(grp, costs[g0:g0 + MAX_LANES], model, W)
            gs = torch.zeros((4 * W, n_chunks), dtype=torch.int64, device=dev)
            _lib.call("mp_score_u8", _lib.ptr(planes), stride, 0, b - a, model.L, model.K, _lib.ptr(bounds), n_chunks,
                      _lib.ptr(tables), W, max_p, _lib.ptr(gs), sh)
            pk.sums[g0:g0 + len(grp)].copy_(gs[:len(grp)])
    pk.allreduce(group)
    counts = pk.counts.cpu().numpy()
    sums = pk.sums.cpu().numpy()
    tokens = np.diff(chunk_bounds_even(n_tokens, n_chunks))
    freq = frequencies_from_counts(counts, n_tokens, model.K)
    return freq, [report_from_sums(sums[i], tokens, getattr(p, "label", "")) for i, p in enumerate(placements)]
