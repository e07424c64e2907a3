"""Token-sharded multi-GPU evaluation.

The token dimension shards naturally: rank r owns tokens [r*N/G, (r+1)*N/G) of the trace (a
contiguous range that may cut through chunks), generates them in place (the generator is
counter-based, so a shard is bit-identical to the same tokens of the full trace), runs the fused
statistics+scoring pass, and the per-rank integer partials — the [L, E] load counts and the
[P, C] per-chunk hop sums, packed into ONE int64 buffer — are summed once: on GPUs by our own
peer-memory kernel over NVLink/NVSwitch (``PeerSum``, NVLS multimem reduction when available), else
with ``torch.distributed.all_reduce`` (gloo works for host tensors).
Integer sums are exact for any world size and any partition, so every rank ends with the same
bits as a single-GPU run; the report floats are then derived once, identically everywhere.
"""
from __future__ import annotations

import os
from typing import Optional, Sequence

import numpy as np

from .errors import ConfigError


def shard_range(n_tokens: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous token range of ``rank``: [floor(r*N/G), floor((r+1)*N/G))."""
    if world < 1 or not 0 <= rank < world:
        raise ConfigError(f"bad rank {rank} for world size {world}")
    return (rank * n_tokens) // world, ((rank + 1) * n_tokens) // world


class PeerSum:
    """Sum of an int64 vector over the ranks of an NCCL group through NVLink / NVSwitch peer memory
    (``mp_allreduce_peers_i64``): the inputs live in symmetric memory
    (``torch.distributed._symmetric_memory``), two halves used on alternate calls, and on a box with
    a multicast object ONE ``multimem.ld_reduce`` per element returns the world's sum from the switch
    (else P2P loads of the peers' copies).  Usage per call: ``b = ps.input()`` (zeroed, this call's
    half), write the partials into ``b``, ``out = ps.allreduce()``.  ``PeerSum.create`` returns None
    where symmetric memory is unavailable (CPU / gloo groups); callers then use
    ``torch.distributed.all_reduce``."""

    _cache: dict = {}
    _epochs: dict = {}  # per group: every call on the group takes the next epoch, whatever its PeerSum

    def __init__(self, n: int, group):
        import torch
        import torch.distributed._symmetric_memory as symm

        from . import _lib
        self.n = n
        self.sym = symm.empty(2 * n, dtype=torch.int64, device="cuda")
        self.hdl = symm.rendezvous(self.sym, group.group_name)
        self.rank, self.world = self.hdl.rank, self.hdl.world_size
        mc = int(getattr(self.hdl, "multicast_ptr", 0) or 0)
        if os.environ.get("MOEPLACE_PEER_NO_MULTICAST"):  # exercise the P2P-load path on an NVLS box
            mc = 0
        dev_ptrs = lambda xs: torch.tensor(xs, dtype=torch.int64, device="cuda")  # noqa: E731 (< 2^63)
        self.peers = [dev_ptrs([p + h * n * 8 for p in self.hdl.buffer_ptrs]) for h in (0, 1)]
        self.mcs = [mc + h * n * 8 if mc else 0 for h in (0, 1)]
        self.pads = dev_ptrs(self.hdl.signal_pad_ptrs)
        self.out = torch.zeros(n, dtype=torch.int64, device="cuda")
        self.err = _lib.new_err()
        self.group_name = group.group_name
        self.epoch = 0  # calls made on this buffer (selects the input half)

    @classmethod
    def create(cls, n: int, group=None):
        import torch.distributed as dist
        try:
            import torch.distributed._symmetric_memory  # noqa: F401
        except ImportError:
            return None
        if not (dist.is_available() and dist.is_initialized()):
            return None
        group = group or dist.group.WORLD
        if dist.get_world_size(group) < 2 or dist.get_backend(group) != "nccl":
            return None
        if n > (1 << 21) // dist.get_world_size(group):  # mp_allreduce_peers_i64's signal-pad budget
            return None
        key = (group.group_name, n)
        if key not in cls._cache:
            try:
                cls._cache[key] = cls(n, group)
            except Exception as e:  # noqa: BLE001 -- no symmetric memory / P2P on this box: NCCL instead
                import sys
                print(f"PeerSum: symmetric memory unavailable ({type(e).__name__}: {e}); using NCCL all_reduce",
                      file=sys.stderr)
                cls._cache[key] = None
        return cls._cache[key]

    def input(self):
        """This call's input half (zeroed): the half of epoch + 1."""
        h = (self.epoch + 1) & 1
        b = self.sym[h * self.n:(h + 1) * self.n]
        b.zero_()
        return b

    def allreduce(self):
        """out <- sum over the group of every rank's current input half (stream-ordered; every rank
        calls it once per input())."""
        from . import _lib
        self.epoch += 1
        h = self.epoch & 1
        ge = PeerSum._epochs.get(self.group_name, 0) + 1  # unique per group: signal pads may be shared
        PeerSum._epochs[self.group_name] = ge
        _lib.call("mp_allreduce_peers_i64", _lib.ptr(self.out), self.n, self.mcs[h] or None, _lib.ptr(self.peers[h]),
                  _lib.ptr(self.pads), self.rank, self.world, ge & 0xFFFFFFFF, _lib.ptr(self.err),
                  _lib.stream_handle())
        return self.out

    def check(self):
        from . import _lib
        _lib.check_err(self.err, "mp_allreduce_peers_i64: a peer did not arrive")


class Packed:
    """One int64 buffer holding [counts (L*E) | hop sums (P*C)]: a single collective per pass.  On an
    NCCL group it lives in symmetric memory and is summed over NVLink/NVSwitch by our own kernel
    (``PeerSum``); otherwise ``torch.distributed.all_reduce`` sums it."""

    def __init__(self, L: int, E: int, P: int, C: int, device=None, group=None):
        import torch
        self.L, self.E, self.P, self.C = L, E, P, C
        self.peer = PeerSum.create(L * E + P * C, group) if device is not None and str(device).startswith("cuda") else None
        self.buf = self.peer.input() if self.peer is not None else torch.zeros(L * E + P * C, dtype=torch.int64,
                                                                                device=device)

    @property
    def counts(self):
        return self.buf[: self.L * self.E].view(self.L, self.E)

    @property
    def sums(self):
        return self.buf[self.L * self.E:].view(self.P, self.C)

    def allreduce(self, group=None) -> "Packed":
        import torch.distributed as dist
        if self.peer is not None:
            self.buf = self.peer.allreduce()  # the sums land in the rank's private buffer
        elif dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=group)
        return self


def sharded_evaluate(model, zipf_s: float, n_tokens: int, n_chunks: int, seed: int,
                     placements: Sequence, costs, group=None, rank: Optional[int] = None,
                     world: Optional[int] = None):
    """Generate this rank's shard on its GPU, build the load counts and the per-chunk hop sums of
    every placement (``costs``: one CostMatrix or one per placement — several topologies can be
    mixed), all-reduce ONE packed int64 buffer, and return the global
    (FrequencyTable, [EvalReport]) — identical on every rank and to a one-GPU run.
    The first 16 placements (32 where the count-contract kernel runs) ride the fused statistics
    pass; further ones are scored 16 (32) per pass."""
    import torch
    import torch.distributed as dist

    from . import _lib
    from .eval import _as_costs, _group_tables, _lanes_for, pass_lanes, report_from_sums
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
    pk = Packed(model.L, model.E, P, n_chunks, dev, group)
    if b > a:
        planes, stride = tr.planes, tr.planes.shape[1]
        bounds = _lib.to_dev(tr.chunk_bounds, torch.int64)
        err = _lib.new_err()
        sh = _lib.stream_handle()
        hl = pass_lanes(tr, costs, hist=True)  # 32 on the count-contract kernel (long chunks), else 16
        head = placements[:hl]
        W = _lanes_for(len(head))
        tables, max_p = _group_tables(head, costs[:hl], model, W)
        sums = torch.zeros((4 * W, n_chunks), dtype=torch.int64, device=dev)
        _lib.call("mp_hist_score_ex_u8", _lib.ptr(planes), stride, 0, b - a, model.L, model.K, model.E,
                  _lib.ptr(bounds), n_chunks, _lib.ptr(tables), W, max_p, _lib.ptr(pk.counts), _lib.ptr(sums),
                  _lib.ptr(err), 0, sh)
        _lib.check_err(err, "sharded_evaluate")
        pk.sums[:len(head)].copy_(sums[:len(head)])
        lanes = pass_lanes(tr, costs)
        for g0 in range(hl, P, lanes):
            grp = placements[g0:g0 + lanes]
            W = _lanes_for(len(grp))
            tables, max_p = _group_tables(grp, costs[g0:g0 + lanes], model, W)
            gs = torch.zeros((4 * W, n_chunks), dtype=torch.int64, device=dev)
            _lib.call("mp_score_u8", _lib.ptr(planes), stride, 0, b - a, model.L, model.K, _lib.ptr(bounds), n_chunks,
                      _lib.ptr(tables), W, max_p, _lib.ptr(gs), sh)
            pk.sums[g0:g0 + len(grp)].copy_(gs[:len(grp)])
    pk.allreduce(group)
    if pk.peer is not None:
        pk.peer.check()
    counts = pk.counts.cpu().numpy()
    sums = pk.sums.cpu().numpy()
    tokens = np.diff(chunk_bounds_even(n_tokens, n_chunks))
    freq = frequencies_from_counts(counts, n_tokens, model.K)
    return freq, [report_from_sums(sums[i], tokens, getattr(p, "label", "")) for i, p in enumerate(placements)]
