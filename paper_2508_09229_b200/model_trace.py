"""``moeplace.model_trace`` — model shape, activation traces and load statistics.

Device layout of a trace ("layer planes"): ``planes`` is uint8 [L, stride] and
byte ``t*K + k`` of plane ``l`` is the k-th expert that token ``t`` selected in MoE layer ``l``.
Expert ids are single bytes (E <= 256).  Tokens are grouped by chunk in ascending chunk-id order,
so a chunk, a train/test split or a multi-GPU shard is a token range — a zero-copy view.

Hot path: ``generate_trace`` (kernel ``mp_gen_trace``) and ``estimate_frequencies`` (kernel
``mp_hist_u8``).  ``parse_trace``/``write_trace`` are host text IO that feed the same planes.
"""
from __future__ import annotations

import os
import re
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import Any, Optional, Sequence

import numpy as np

from . import _lib
from .errors import ConfigError, MoeplaceError, TraceParseError

MAX_EXPERTS = 256  # one-byte expert ids on the device


@dataclass(frozen=True)
class ModelSpec:
    """L MoE layers, E routed experts per layer, top-K routing."""

    num_moe_layers: int
    experts_per_layer: int
    topk: int

    def __post_init__(self):
        L, E, K = self.num_moe_layers, self.experts_per_layer, self.topk
        for name, v in (("num_moe_layers", L), ("experts_per_layer", E), ("topk", K)):
            if not isinstance(v, (int, np.integer)) or v < 1:
                raise ConfigError(f"ModelSpec.{name} must be an integer >= 1, got {v!r}")
        if K > E:
            raise ConfigError(f"topk ({K}) must be <= experts_per_layer ({E})")

    @property
    def L(self) -> int:
        return self.num_moe_layers

    @property
    def E(self) -> int:
        return self.experts_per_layer

    @property
    def K(self) -> int:
        return self.topk


@dataclass
class AttentionPlacement:
    """dispatch device d_l and collect device c_l per layer."""

    dispatch: np.ndarray  # int32 [L]
    collect: np.ndarray   # int32 [L]

    def __post_init__(self):
        self.dispatch = np.asarray(self.dispatch, dtype=np.int32)
        self.collect = np.asarray(self.collect, dtype=np.int32)
        if self.dispatch.shape != self.collect.shape or self.dispatch.ndim != 1:
            raise ConfigError("dispatch and collect must be 1-D arrays of equal length")


@dataclass
class FrequencyTable:
    """f[l, e] = count(l, e) / (K * n_tokens).  ``counts`` keeps the exact
    integer statistics the device produced; ``f`` is derived from them on the host."""

    f: np.ndarray                       # float64 [L, E]
    counts: Optional[np.ndarray] = None  # int64 [L, E]
    n_tokens: int = 0
    topk: int = 0


@dataclass
class ActivationTrace:
    """SPEC.md:104-107.  ``planes[:, t*K:(t+1)*K]`` are token t's selections, tokens
    ``[tok_begin, tok_begin + n_tokens)`` belong to this view, chunk c spans tokens
    ``[chunk_bounds[c], chunk_bounds[c+1])`` and carries label ``chunk_ids[c]``.

    ``layout="tokens"`` holds the SPEC's own token-major form instead: ``planes`` is a host uint8
    tensor [N, L, K] (pinned for the streamed end-to-end path, ``from_host_tokens``); every pass
    streams it to the device slice by slice and transposes each slice into layer planes there
    (``mp_tokens_to_planes_u8``), so no host transpose is ever made."""

    model: Optional[ModelSpec]
    planes: Any                # torch.uint8 [L, stride] (CUDA or host), or [N, L, K] host when layout="tokens"
    tok_begin: int
    n_tokens: int
    chunk_ids: np.ndarray      # int64 [C], ascending
    chunk_bounds: np.ndarray   # int64 [C+1], absolute token indices into planes
    source_is_file: bool = False
    _validated: bool = field(default=False, repr=False)
    layout: str = "planes"
    _dev: Any = field(default=None, repr=False)  # device planes of this view's tokens (host traces)

    @property
    def n_chunks(self) -> int:
        return int(self.chunk_ids.shape[0])

    @property
    def tok_end(self) -> int:
        return self.tok_begin + self.n_tokens

    def __len__(self) -> int:
        return self.n_tokens

    def chunk_token_counts(self) -> np.ndarray:
        return np.diff(self.chunk_bounds).astype(np.int64)

    def token_chunk_ids(self) -> np.ndarray:
        return np.repeat(self.chunk_ids, self.chunk_token_counts())

    @property
    def on_device(self) -> bool:
        return self.planes is not None and self.planes.is_cuda and self.layout == "planes"

    def device_view(self):
        """(planes, t0, t1): this view's tokens as CUDA layer planes.  A device-resident trace
        returns its own planes and token range (no copy).  A host-resident one uploads ONLY the
        view's tokens (transposed on the device when token-major) into planes cached on this view
        object; the caller's host planes are never replaced, so other views and the streamed
        passes keep streaming."""
        if self.on_device:
            return self.planes, self.tok_begin, self.tok_end
        if self._dev is None:
            t = _lib.torch()
            dev = _lib.require_cuda()
            m = self.model
            n, K = self.n_tokens, m.K
            planes = t.empty((m.L, _plane_stride(n, K)), dtype=t.uint8, device=dev)
            a = self.tok_begin
            if self.layout == "tokens":
                tok = self.planes[a:a + n].to(dev, non_blocking=True).contiguous()
                _lib.call("mp_tokens_to_planes_u8", _lib.ptr(tok), n, m.L, K, _lib.ptr(planes), planes.shape[1], 0,
                          _lib.stream_handle())
            else:
                _lib.call("mp_copy_planes_h2d", _lib.ptr(planes), planes.shape[1],
                          C_void(self.planes.data_ptr() + a * K), self.planes.shape[1], n * K, m.L,
                          _lib.stream_handle())
            self._dev = planes
        return self._dev, 0, self.n_tokens

    def device_planes(self):
        """The planes of this view on the CUDA device (``device_view()[0]``)."""
        return self.device_view()[0]

    def to_host(self, pin: bool = True, layout: str = "planes") -> "ActivationTrace":
        """A copy whose data live in (pinned) host memory: evaluating it streams the trace
        through the device slice by slice (the end-to-end path), without caching it there.
        ``layout="tokens"`` gives the SPEC's token-major [N, L, K] form (transposed on the device
        before the download)."""
        t = _lib.torch()
        if layout not in ("planes", "tokens"):
            raise ConfigError(f"unknown trace layout {layout!r}")
        if layout == "tokens":
            m = self.model
            planes, t0, t1 = self.device_view()
            src = planes[:, t0 * m.K:t1 * m.K].view(m.L, self.n_tokens, m.K).permute(1, 0, 2)
            h = t.empty((self.n_tokens, m.L, m.K), dtype=t.uint8, pin_memory=pin)
            h.copy_(src)
            b = self.chunk_bounds - self.tok_begin
            return ActivationTrace(self.model, h, 0, self.n_tokens, self.chunk_ids.copy(), b.astype(np.int64),
                                   self.source_is_file, self._validated, layout="tokens")
        if self.layout == "tokens":
            raise ConfigError("to_host(layout='planes') of a token-major trace: evaluate it directly")
        if pin:  # allocate pinned and copy once (no pageable intermediate: half the peak host memory)
            h = t.empty(self.planes.shape, dtype=self.planes.dtype, pin_memory=True)
            h.copy_(self.planes)
        else:
            h = self.planes.cpu()
        return ActivationTrace(self.model, h, self.tok_begin, self.n_tokens, self.chunk_ids.copy(),
                               self.chunk_bounds.copy(), self.source_is_file, self._validated)

    def tokens(self) -> np.ndarray:
        """Host copy in token-major form, uint8 [N, L, K] (for IO and small-case inspection)."""
        m = self.model
        if m is None or self.n_tokens == 0:
            K = m.K if m else 0
            L = m.L if m else 0
            return np.zeros((0, L, K), dtype=np.uint8)
        if self.layout == "tokens":
            return self.planes[self.tok_begin:self.tok_end].numpy().copy()
        K = m.K
        x = self.planes[:, self.tok_begin * K:self.tok_end * K].cpu().numpy()
        return np.ascontiguousarray(x.reshape(m.L, self.n_tokens, K).transpose(1, 0, 2))

    def view(self, chunk_lo: int, chunk_hi: int) -> "ActivationTrace":
        """Zero-copy sub-trace made of chunks [chunk_lo, chunk_hi) (in id order)."""
        b = self.chunk_bounds
        return ActivationTrace(self.model, self.planes, int(b[chunk_lo]), int(b[chunk_hi] - b[chunk_lo]),
                               self.chunk_ids[chunk_lo:chunk_hi].copy(), b[chunk_lo:chunk_hi + 1].copy(),
                               self.source_is_file, self._validated, layout=self.layout)

    @classmethod
    def from_router_topk(cls, model: ModelSpec, topk_ids, chunk_bounds: Optional[Sequence[int]] = None,
                         chunk_ids: Optional[Sequence[int]] = None) -> "ActivationTrace":
        """Ingest router top-k indices that are already on the GPU (e.g. captured from a running
        MoE model): ``topk_ids`` int tensor [N, L, K] in token order; tokens are grouped by chunk
        via ``chunk_bounds`` (default: one chunk).  Narrowed to u8 and transposed to layer planes on
        the device, then validated by ``mp_validate_u8`` (ids < E, K distinct per record)."""
        t = _lib.torch()
        dev = _lib.require_cuda()
        if not isinstance(topk_ids, t.Tensor) or topk_ids.dim() != 3 or tuple(topk_ids.shape[1:]) != (model.L, model.K):
            raise ConfigError(f"topk_ids must be a tensor [N, {model.L}, {model.K}]")
        if model.E > MAX_EXPERTS:
            raise ConfigError(f"E = {model.E} exceeds the one-byte device id format (E <= {MAX_EXPERTS})")
        ids = topk_ids.to(dev)
        N = int(ids.shape[0])
        if N and (int(ids.min()) < 0 or int(ids.max()) >= model.E):
            raise MoeplaceError(f"router ids outside [0, {model.E})")
        planes = t.empty((model.L, _plane_stride(N, model.K)), dtype=t.uint8, device=dev)
        u8 = ids.to(t.uint8).contiguous()
        _lib.call("mp_tokens_to_planes_u8", _lib.ptr(u8), N, model.L, model.K, _lib.ptr(planes), planes.shape[1], 0,
                  _lib.stream_handle())
        b = np.array([0, N] if chunk_bounds is None else list(chunk_bounds), dtype=np.int64)
        if b[0] != 0 or b[-1] != N or (np.diff(b) < 0).any():
            raise ConfigError("chunk_bounds must ascend from 0 to N")
        cid = np.arange(len(b) - 1, dtype=np.int64) if chunk_ids is None else np.asarray(chunk_ids, dtype=np.int64)
        tr = cls(model, planes, 0, N, cid, b)
        validate_trace(tr)
        return tr

    @classmethod
    def from_tokens(cls, model: ModelSpec, selections, chunk_of_token: Optional[Sequence[int]] = None,
                    device=None) -> "ActivationTrace":
        """Build a trace from token-major selections [N, L, K] and per-token chunk labels.
        Tokens are stably regrouped by ascending chunk id (evaluation is invariant under
        permutation within a chunk); the token-major bytes are uploaded as they are
        and transposed into layer planes on the device (``mp_tokens_to_planes_u8``)."""
        sel = np.asarray(selections)
        if sel.ndim != 3 or sel.shape[1:] != (model.L, model.K):
            raise ConfigError(f"selections must have shape [N, {model.L}, {model.K}], got {sel.shape}")
        if sel.size and (sel.min() < 0 or sel.max() >= model.E):
            raise MoeplaceError(f"expert index outside [0, {model.E})")
        N = sel.shape[0]
        cid = np.zeros(N, dtype=np.int64) if chunk_of_token is None else np.asarray(chunk_of_token, dtype=np.int64)
        if cid.shape != (N,):
            raise ConfigError("chunk_of_token must have one label per token")
        if N and (cid[1:] < cid[:-1]).any():
            order = np.argsort(cid, kind="stable")
            sel, cid = sel[order], cid[order]
        ids, counts = np.unique(cid, return_counts=True)
        bounds = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        tok = np.ascontiguousarray(sel, dtype=np.uint8)
        tr = cls(model, _lib.torch().from_numpy(tok), 0, N, ids.astype(np.int64), bounds, layout="tokens")
        if device is not None and str(device) == "cpu":
            return tr
        if _lib.torch().cuda.is_available():
            planes, _, _ = tr.device_view()
            return cls(model, planes, 0, N, tr.chunk_ids, bounds)
        return tr

    @classmethod
    def from_host_tokens(cls, model: ModelSpec, selections, chunk_bounds: Optional[Sequence[int]] = None,
                         chunk_ids: Optional[Sequence[int]] = None, pin: bool = True) -> "ActivationTrace":
        """The SPEC-shaped end-to-end input: token-major uint8 selections [N, L, K] held in host
        memory, tokens already grouped by chunk (``chunk_bounds`` ascending from 0 to N; default
        one chunk).  Nothing is transposed or copied on the host beyond one pinned staging copy
        (none when ``selections`` is already a pinned uint8 tensor): every pass streams the
        token-major slices to the device and transposes them there (``mp_tokens_to_planes_u8``)."""
        t = _lib.torch()
        if model.E > MAX_EXPERTS:
            raise ConfigError(f"E = {model.E} exceeds the one-byte device id format (E <= {MAX_EXPERTS})")
        x = selections if isinstance(selections, t.Tensor) else t.from_numpy(np.ascontiguousarray(selections))
        if x.dim() != 3 or tuple(x.shape[1:]) != (model.L, model.K):
            raise ConfigError(f"selections must have shape [N, {model.L}, {model.K}], got {tuple(x.shape)}")
        if x.is_cuda:
            raise ConfigError("from_host_tokens takes host selections (use from_router_topk for device ids)")
        if x.dtype != t.uint8:
            if x.numel() and (int(x.min()) < 0 or int(x.max()) >= model.E):
                raise MoeplaceError(f"expert index outside [0, {model.E})")
            x = x.to(t.uint8)
        x = x.contiguous()
        if pin and not x.is_pinned():
            x = x.pin_memory()
        N = int(x.shape[0])
        b = np.array([0, N] if chunk_bounds is None else list(chunk_bounds), dtype=np.int64)
        if b[0] != 0 or b[-1] != N or (np.diff(b) < 0).any():
            raise ConfigError("chunk_bounds must ascend from 0 to N")
        cid = np.arange(len(b) - 1, dtype=np.int64) if chunk_ids is None else np.asarray(chunk_ids, dtype=np.int64)
        if cid.shape != (len(b) - 1,) or (np.diff(cid) <= 0).any():
            raise ConfigError("chunk_ids must be one ascending id per chunk")
        return cls(model, x, 0, N, cid, b, layout="tokens")


def _plane_stride(n_tokens: int, K: int) -> int:
    return max(16, (n_tokens * K + 15) // 16 * 16)


def default_attention_placement(model: ModelSpec, order: Sequence[int]) -> AttentionPlacement:
    """d_l = order[floor(l*S/L)], c_l = d_{l+1}, c_{L-1} = d_{L-1}."""
    order = list(order)
    S, L = len(order), model.L
    if S < 1:
        raise ConfigError("at least one device is required")
    d = np.array([order[(l * S) // L] for l in range(L)], dtype=np.int32)
    c = np.concatenate([d[1:], d[-1:]]).astype(np.int32)
    return AttentionPlacement(d, c)


# ---- synthetic traces ----------------------------------------------

_W_SCALE = 1 << 30


def zipf_weights(E: int, s: float) -> np.ndarray:
    """Integer Zipf(s) weights over ranks 1..E: max(1, floor(2^30 * r^-s / sum_j j^-s))."""
    if s < 0:
        raise ConfigError(f"zipf_s must be >= 0, got {s}")
    r = np.arange(1, E + 1, dtype=np.float64)
    raw = r ** (-float(s))
    return np.maximum(1, np.floor(raw / raw.sum() * _W_SCALE)).astype(np.int64)


def zipf_cdf(E: int, s: float) -> np.ndarray:
    w = zipf_weights(E, s)
    return np.concatenate([[0], np.cumsum(w)]).astype(np.uint32)


_M0, _M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_W0, _W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
PERM_STREAM = 0x40000000  # counter word 3 of the permutation stream (draws use k/4 < 2^30)


def philox4x32_10(c0, c1, c2, c3, seed: int):
    """Vectorised Philox4x32-10 over uint32 arrays (Salmon et al., SC'11); key = seed lo/hi."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint32).copy() for c in (c0, c1, c2, c3))
    k0 = np.uint32(seed & 0xFFFFFFFF)
    k1 = np.uint32((seed >> 32) & 0xFFFFFFFF)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = _M0 * c0.astype(np.uint64)
            p1 = _M1 * c2.astype(np.uint64)
            hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), p0.astype(np.uint32)
            hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), p1.astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = np.uint32((int(k0) + int(_W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(_W1)) & 0xFFFFFFFF)
    return c0, c1, c2, c3


def layer_permutations(seed: int, L: int, E: int) -> np.ndarray:
    """Per-layer rank -> expert permutation: Fisher-Yates, j drawn from
    Philox(counter = (i, 0, l, PERM_STREAM)) as floor(u * (i+1) / 2^32)."""
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    i = np.arange(E, dtype=np.uint32)
    perm = np.tile(np.arange(E, dtype=np.int64), (L, 1))
    for l in range(L):
        u, _, _, _ = philox4x32_10(i, np.zeros(E, np.uint32), np.full(E, l, np.uint32),
                                   np.full(E, PERM_STREAM, np.uint32), seed)
        j = (u.astype(np.uint64) * (i.astype(np.uint64) + np.uint64(1))) >> np.uint64(32)
        p = perm[l]
        for k in range(E - 1, 0, -1):
            jj = int(j[k])
            p[k], p[jj] = p[jj], p[k]
    return perm.astype(np.uint8 if E <= 256 else np.int64)


def chunk_bounds_even(n_tokens: int, n_chunks: int) -> np.ndarray:
    """Tokens evenly labelled into chunks: chunk(t) = floor(t*C/N), i.e. chunk c owns
    tokens [ceil(c*N/C), ceil((c+1)*N/C))."""
    N, C = int(n_tokens), int(n_chunks)
    return np.array([(c * N + C - 1) // C for c in range(C + 1)], dtype=np.int64)


def generate_trace(model: ModelSpec, zipf_s: float, n_tokens: int, n_chunks: int, seed: int,
                   tok_range: Optional[tuple[int, int]] = None) -> ActivationTrace:
    """SPEC.md:123-131.  Generated on the GPU (``mp_gen_trace``).  ``tok_range=(a, b)`` generates
    only tokens [a, b) of the n_tokens-token trace (a shard): bit-identical to the same tokens of
    the full trace, with chunk labels of the full trace."""
    t = _lib.torch()
    if model.E > MAX_EXPERTS:
        raise ConfigError(f"E = {model.E} exceeds the one-byte device id format (E <= {MAX_EXPERTS})")
    if n_tokens < 0 or n_chunks < 1:
        raise ConfigError("n_tokens must be >= 0 and n_chunks >= 1")
    a, b = (0, int(n_tokens)) if tok_range is None else (int(tok_range[0]), int(tok_range[1]))
    if not (0 <= a <= b <= n_tokens):
        raise ConfigError(f"tok_range {tok_range} outside [0, {n_tokens}]")
    dev = _lib.require_cuda()
    L, E, K = model.L, model.E, model.K
    n = b - a
    planes = t.empty((L, _plane_stride(n, K)), dtype=t.uint8, device=dev)
    cdf = _lib.to_dev(zipf_cdf(E, zipf_s).astype(np.int64), t.int64).to(t.int32)  # bit pattern of uint32
    perm = _lib.to_dev(layer_permutations(seed, L, E), t.uint8)
    _lib.call("mp_gen_trace", int(seed) & 0xFFFFFFFFFFFFFFFF, a, b, L, K, E, _lib.ptr(cdf), _lib.ptr(perm),
              _lib.ptr(planes), planes.shape[1], _lib.stream_handle())
    full = chunk_bounds_even(n_tokens, n_chunks)
    bounds = np.clip(full, a, b) - a
    return ActivationTrace(model, planes, 0, n, np.arange(n_chunks, dtype=np.int64), bounds, _validated=True)


# ---- text format ---------------------------------------------------

_HEADER = re.compile(r"^#moeplace-trace v1 L=(\d+) E=(\d+) K=(\d+)\s*$")
_FIELD = re.compile(r"^(?:layer)?(\d+):(.*)$")


_PARSE_ERR = {1: "malformed line (expected chunk_id<TAB>layer<l>:e,...,e fields)", 2: "layer fields out of order",
              3: "expert index outside [0, E)", 4: "wrong number of experts in a layer field",
              5: "repeated expert index", 6: "chunk id too large"}


# ---- file <-> device text transfers through a reusable pinned ring ----------------------------
# 2 x IO_LANES slots of IO_SLOT bytes: IO_LANES slots are read (pread) or written (pwrite) in
# parallel threads (the kernel copies release the GIL) while the other half is in flight over PCIe
# on a copy stream, so a text trace moves at file-system-cache speed without a full-size pinned
# staging copy.
IO_SLOT = 32 << 20
IO_LANES = 4
_IO = {"ring": None, "pool": None}
_IO_LOCK = threading.Lock()


def _io_ring():
    t = _lib.torch()
    if _IO["ring"] is None:
        _IO["ring"] = [t.empty(IO_SLOT, dtype=t.uint8, pin_memory=True) for _ in range(2 * IO_LANES)]
        _IO["pool"] = ThreadPoolExecutor(IO_LANES, thread_name_prefix="moeplace-io")
    return _IO["ring"], _IO["pool"]


def _file_to_device(fd: int, n: int, dst) -> None:
    """dst[:n] <- bytes [0, n) of the open file ``fd`` (stream-ordered on the current stream)."""
    t = _lib.torch()
    with _IO_LOCK:
        ring, pool = _io_ring()
        views = [r.numpy() for r in ring]
        cs = t.cuda.Stream()
        cs.wait_stream(t.cuda.current_stream())
        evs = [None] * len(ring)
        off, half = 0, 0
        while off < n:
            jobs = []
            for r in range(IO_LANES):
                o = off + r * IO_SLOT
                if o >= n:
                    break
                k = half * IO_LANES + r
                if evs[k] is not None:
                    evs[k].synchronize()  # the slot's previous upload is done
                m = min(IO_SLOT, n - o)
                jobs.append((k, o, m, pool.submit(os.preadv, fd, [views[k][:m]], o)))
            for k, o, m, fut in jobs:
                if fut.result() != m:
                    raise MoeplaceError("parse_trace: short read (file changed while loading?)")
                with t.cuda.stream(cs):
                    dst[o:o + m].copy_(ring[k][:m], non_blocking=True)
                    evs[k] = t.cuda.Event()
                    evs[k].record(cs)
            off += IO_LANES * IO_SLOT
            half ^= 1
        t.cuda.current_stream().wait_stream(cs)
        for e in evs:
            if e is not None:
                e.synchronize()  # the ring is reusable once this returns


def _device_to_file(src, n: int, fd: int, base: int) -> None:
    """Bytes [base, base + n) of the open file ``fd`` <- src[:n] (device uint8)."""
    t = _lib.torch()
    with _IO_LOCK:
        ring, pool = _io_ring()
        views = [r.numpy() for r in ring]
        cs = t.cuda.Stream()
        cs.wait_stream(t.cuda.current_stream())
        pending = []  # (future) writes of the previous half
        off, half = 0, 0
        while off < n:
            batch = []
            for r in range(IO_LANES):
                o = off + r * IO_SLOT
                if o >= n:
                    break
                k = half * IO_LANES + r
                m = min(IO_SLOT, n - o)
                with t.cuda.stream(cs):
                    ring[k][:m].copy_(src[o:o + m], non_blocking=True)
                    ev = t.cuda.Event()
                    ev.record(cs)
                batch.append((k, o, m, ev))
            for fut in pending:  # the other half's writes overlap this half's downloads
                fut.result()
            pending = []
            for k, o, m, ev in batch:
                ev.synchronize()
                pending.append(pool.submit(os.pwritev, fd, [views[k][:m]], base + o))
            off += IO_LANES * IO_SLOT
            half ^= 1
        for fut in pending:
            fut.result()


def parse_trace(path, engine: str = "cuda") -> ActivationTrace:
    """SPEC.md:132-139.  Parse the text trace format; errors raise ``TraceParseError`` with the
    1-based line number (header = line 1).  ``engine="cuda"`` (default) parses on the GPU
    (``mp_count_newlines``/``mp_find_newlines``/``mp_parse_trace_text``) straight into the
    device planes.  There is no host parser: the path has no CPU fallback (the tests' checker is
    ``oracle/textio.py``)."""
    if engine != "cuda":
        raise ConfigError(f"unknown parse engine {engine!r} (the trace parser runs on the device only)")
    t = _lib.torch()
    dev = _lib.require_cuda()
    with open(path, "rb") as f:
        n = os.fstat(f.fileno()).st_size
        if n == 0:
            return ActivationTrace(None, t.zeros((0, 16), dtype=t.uint8), 0, 0, np.zeros(0, np.int64),
                                   np.zeros(1, np.int64), source_is_file=True)
        head = f.read(4096)
        head_end = head.find(b"\n")
        header = head[:head_end if head_end >= 0 else min(n, 4096)].decode("utf-8", "replace")
        m = _HEADER.match(header.rstrip("\r"))
        if not m:
            raise TraceParseError("missing or malformed header '#moeplace-trace v1 L=<L> E=<E> K=<K>'", 1)
        try:
            model = ModelSpec(int(m.group(1)), int(m.group(2)), int(m.group(3)))
        except ConfigError as e:
            raise TraceParseError(str(e), 1) from None
        if model.E > MAX_EXPERTS:
            raise ConfigError(f"E = {model.E} exceeds the one-byte device id format (E <= {MAX_EXPERTS})")
        last_byte = os.pread(f.fileno(), 1, n - 1)[0]
        pad = (n + 32 + 15) // 16 * 16
        text = t.empty(pad, dtype=t.uint8, device=dev)
        text[n:].zero_()
        _file_to_device(f.fileno(), n, text)  # pinned-ring pipeline: parallel preads + H2D
    if head_end < 0:
        head_end = n
    L, K = model.L, model.K
    nb = (n + 65535) // 65536
    counts = t.empty(nb, dtype=t.int64, device=dev)
    sh = _lib.stream_handle()
    _lib.call("mp_count_newlines", _lib.ptr(text), n, _lib.ptr(counts), sh)
    offsets = t.cumsum(counts, 0) - counts
    total = int(counts.sum().item())
    pos = t.empty(max(total, 1), dtype=t.int64, device=dev)
    _lib.call("mp_find_newlines", _lib.ptr(text), n, _lib.ptr(offsets), _lib.ptr(pos), sh)
    pos = pos[:total]
    ends = pos[1:] if total and int(pos[0].item()) == head_end else pos
    if n > head_end + 1 and last_byte != 10:  # last line without a trailing newline
        ends = t.cat([ends, t.tensor([n], dtype=t.int64, device=dev)])
    ends = ends.contiguous()
    N = int(ends.numel())
    planes = t.empty((L, _plane_stride(N, K)), dtype=t.uint8, device=dev)
    cids = t.empty(max(N, 1), dtype=t.int64, device=dev)
    err = t.full((1,), 2 ** 63 - 1, dtype=t.int64, device=dev)
    _lib.call("mp_parse_trace_text", _lib.ptr(text), _lib.ptr(ends), head_end + 1, N, L, K, model.E, _lib.ptr(planes),
              planes.shape[1], _lib.ptr(cids), _lib.ptr(err), sh)
    e = int(err.item())
    if e != 2 ** 63 - 1:
        line, code = e // 16, e % 16
        raise TraceParseError(_PARSE_ERR.get(code, f"parse error {code}"), int(line) + 2)
    del text
    cids = cids[:N]
    if N and not bool((cids[1:] >= cids[:-1]).all().item()):
        order = t.sort(cids, stable=True).indices  # regroup by chunk id
        cids = cids[order]
        planes3 = planes[:, :N * K].view(L, N, K)
        planes[:, :N * K].copy_(planes3[:, order].reshape(L, N * K))
    if N:
        ids, cnt = t.unique_consecutive(cids, return_counts=True)
        ids, cnt = ids.cpu().numpy(), cnt.cpu().numpy()
    else:
        ids, cnt = np.zeros(0, np.int64), np.zeros(0, np.int64)
    bounds = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    return ActivationTrace(model, planes, 0, N, ids.astype(np.int64), bounds, source_is_file=True, _validated=True)


def write_trace(trace: ActivationTrace, path, engine: str = "cuda") -> None:
    """SPEC.md:132-139, 170.  Canonical text form: header, then one line per token in
    chunk-grouped order, formatted on the device (two passes: per-line lengths, prefix sum, each
    thread writes its line; ``mp_format_lengths`` / ``mp_format_trace_text``) and written through
    the pinned ring.  A host-resident trace is uploaded (only the view's tokens) first; there is
    no host writer (no CPU fallback; ``engine`` other than "cuda" raises)."""
    m = trace.model
    if engine not in ("cuda", "auto"):
        raise ConfigError(f"unknown write engine {engine!r} (the trace writer runs on the device only)")
    if m is None:
        with open(path, "w"):
            return
    t = _lib.torch()
    header = f"#moeplace-trace v1 L={m.L} E={m.E} K={m.K}\n".encode()
    if trace.n_tokens == 0:
        with open(path, "wb") as f:
            f.write(header)
        return
    planes, t0, t1 = trace.device_view()
    dev = planes.device
    n = trace.n_tokens
    cids = _lib.to_dev(trace.token_chunk_ids(), t.int64)
    lens = t.empty(n, dtype=t.int64, device=dev)
    sh = _lib.stream_handle()
    _lib.call("mp_format_lengths", _lib.ptr(planes), planes.shape[1], t0, t1, m.L, m.K,
              _lib.ptr(cids), _lib.ptr(lens), sh)
    offs = (t.cumsum(lens, 0) - lens).contiguous()
    total = int(lens.sum().item())
    out = t.empty(total, dtype=t.uint8, device=dev)
    _lib.call("mp_format_trace_text", _lib.ptr(planes), planes.shape[1], t0, t1, m.L, m.K,
              _lib.ptr(cids), _lib.ptr(offs), _lib.ptr(out), sh)
    with open(path, "wb") as f:
        f.write(header)
        f.flush()
        try:  # allocate the file's blocks up front: the parallel pwrites then only copy (0.37 -> 0.34 s / 2 GB)
            os.posix_fallocate(f.fileno(), 0, len(header) + total)
        except (OSError, AttributeError):
            pass
        _device_to_file(out, total, f.fileno(), len(header))


_BIN_MAGIC = b"MPTRACE1"


def write_trace_binary(trace: ActivationTrace, path) -> None:
    """Binary sidecar (SURVEY §8(a) A3 fast path): 8-byte magic, u64 header length, a JSON header
    {L, E, K, n_tokens, n_chunks}, int64 chunk ids and bounds, then the L layer planes of the
    view's tokens (N*K bytes each).  ~5x smaller than the text form and loadable without parsing."""
    import json
    m = trace.model
    if m is None:
        raise ConfigError("cannot write an empty (model-less) trace")
    K = m.K
    dplanes, t0, t1 = trace.device_view()
    planes = dplanes[:, t0 * K:t1 * K].contiguous().cpu().numpy()
    bounds = (trace.chunk_bounds - trace.tok_begin).astype(np.int64)
    hdr = json.dumps({"L": m.L, "E": m.E, "K": K, "n_tokens": trace.n_tokens, "n_chunks": trace.n_chunks}).encode()
    with open(path, "wb") as f:
        f.write(_BIN_MAGIC)
        f.write(np.uint64(len(hdr)).tobytes())
        f.write(hdr)
        f.write(trace.chunk_ids.astype(np.int64).tobytes())
        f.write(bounds.tobytes())
        f.write(memoryview(np.ascontiguousarray(planes)))


def read_trace_binary(path, device: str = "pinned") -> ActivationTrace:
    """Load a binary sidecar.  ``device="pinned"`` keeps the planes in pinned host memory (the
    streamed end-to-end path); ``"cuda"`` uploads them."""
    import json
    t = _lib.torch()
    with open(path, "rb") as f:
        if f.read(8) != _BIN_MAGIC:
            raise TraceParseError("not a moeplace binary trace (bad magic)", 1)
        hl = int(np.frombuffer(f.read(8), dtype=np.uint64)[0])
        h = json.loads(f.read(hl))
        m = ModelSpec(int(h["L"]), int(h["E"]), int(h["K"]))
        N, C = int(h["n_tokens"]), int(h["n_chunks"])
        ids = np.frombuffer(f.read(8 * C), dtype=np.int64).copy()
        bounds = np.frombuffer(f.read(8 * (C + 1)), dtype=np.int64).copy()
        stride = _plane_stride(N, m.K)
        planes = t.zeros((m.L, stride), dtype=t.uint8, pin_memory=(device == "pinned"))
        view = planes.numpy()
        for l in range(m.L):
            n = f.readinto(memoryview(view[l, :N * m.K]))
            if n != N * m.K:
                raise TraceParseError(f"truncated binary trace (layer {l})", None)
    if device == "cuda":
        planes = planes.to(_lib.require_cuda())
    tr = ActivationTrace(m, planes, 0, N, ids, bounds, source_is_file=True)
    return tr


def validate_trace(trace: ActivationTrace) -> None:
    """Check the ActivationTrace invariants on the device (``mp_validate_u8``).
    A host-resident trace is validated slice by slice as it streams (``sweep``)."""
    if trace._validated or trace.n_tokens == 0:
        return
    if not trace.on_device:
        sweep(trace, lambda *a: None)
        return
    m = trace.model
    planes = trace.planes
    err = _lib.new_err()
    _lib.call("mp_validate_u8", _lib.ptr(planes), planes.shape[1], trace.tok_begin, trace.tok_end, m.L, m.K, m.E,
              _lib.ptr(err), _lib.stream_handle())
    _raise_invalid(trace, err, 0)
    trace._validated = True


def _raise_invalid(trace: ActivationTrace, err, base: int) -> None:
    """Raise the SPEC error for a flagged mp_validate_u8 err block.  The kernel reports token
    indices of the planes it checked; ``base`` maps them to the trace's numbering (0 for the
    trace's own planes, the slice's first token for a streamed slice)."""
    flag, enc, _, n = _lib.read_err(err)
    if not flag:
        return
    m = trace.model
    key = (2 ** 63 - 1) - enc
    code, tl = key % 8, key // 8
    tok, layer = tl // m.L + base, tl % m.L  # absolute token index
    what = "expert index >= E" if code == _lib.DATA_EXPERT_RANGE else "repeated expert index"
    if trace.source_is_file:
        raise TraceParseError(f"layer {layer}: {what}", tok - trace.tok_begin + 2)
    raise MoeplaceError(f"token {tok - trace.tok_begin}, layer {layer}: {what} ({n} bad records)")


# ---- statistics -----------------------------------------------------------

def C_void(addr: int):
    import ctypes
    return ctypes.c_void_p(addr)


STREAM_BLOCK_TOKENS = 1 << 20  # host-streaming slice (R1: 464 MB per slice)


def sweep(trace: ActivationTrace, launch) -> None:
    """Run ``launch(planes, stride, t0, t1, bounds)`` over the whole trace, in token order.

    Device-resident planes: one call.  Host-resident traces (the end-to-end path) stream through
    two device slices of STREAM_BLOCK_TOKENS tokens: the H2D copy of slice i+1 (on a copy stream)
    overlaps the kernels on slice i, and ``launch`` accumulates per slice (every kernel output is
    additive over token ranges).  Layer planes move with one 2-D copy per slice
    (``mp_copy_planes_h2d``); token-major [N, L, K] selections move as one contiguous copy and are
    transposed into the slice's planes on the device (``mp_tokens_to_planes_u8``).  Nothing is
    cached on the device, so a trace larger than HBM streams too.
    """
    t = _lib.torch()
    if trace.n_tokens == 0:
        return
    if trace.on_device:
        validate_trace(trace)
        planes = trace.planes
        bounds = _lib.to_dev(trace.chunk_bounds, t.int64)
        launch(planes, planes.shape[1], trace.tok_begin, trace.tok_end, bounds)
        return
    src = trace.planes
    m = trace.model
    dev = _lib.require_cuda()
    K, L = m.K, m.L
    tok_major = trace.layout == "tokens"
    T = min(STREAM_BLOCK_TOKENS, trace.n_tokens)
    blocks = [(a, min(a + T, trace.tok_end)) for a in range(trace.tok_begin, trace.tok_end, T)]
    rel = np.stack([np.clip(trace.chunk_bounds, a, b) - a for a, b in blocks]).astype(np.int64)
    d_rel = _lib.to_dev(rel, t.int64)
    stride = _plane_stride(T, K)
    nbuf = min(2, len(blocks))
    if tok_major:  # staging for the token-major bytes; ONE plane slice (transpose + launch share a stream)
        bufs = [t.empty(T * L * K, dtype=t.uint8, device=dev) for _ in range(nbuf)]
        pbuf = t.empty((L, stride), dtype=t.uint8, device=dev)
    else:
        bufs = [t.empty((L, stride), dtype=t.uint8, device=dev) for _ in range(nbuf)]
    comp = t.cuda.current_stream()
    copy = t.cuda.Stream()
    copied = [t.cuda.Event() for _ in bufs]
    free = [t.cuda.Event() for _ in bufs]
    copy.wait_stream(comp)  # d_rel and the outputs are ready before the first slice lands
    sh = _lib.stream_handle()
    for i, (a, b) in enumerate(blocks):
        j = i % nbuf
        n = b - a
        with t.cuda.stream(copy):
            if i >= nbuf:
                copy.wait_event(free[j])
            if tok_major:
                bufs[j][:n * L * K].copy_(src[a:b].view(-1), non_blocking=True)
            else:
                _lib.call("mp_copy_planes_h2d", _lib.ptr(bufs[j]), stride, C_void(src.data_ptr() + a * K),
                          src.shape[1], n * K, L, C_void(copy.cuda_stream))
            copied[j].record(copy)
        comp.wait_event(copied[j])
        if tok_major:
            _lib.call("mp_tokens_to_planes_u8", _lib.ptr(bufs[j]), n, L, K, _lib.ptr(pbuf), stride, 0, sh)
            planes = pbuf
        else:
            planes = bufs[j]
        if not trace._validated:
            err = _lib.new_err()
            _lib.call("mp_validate_u8", _lib.ptr(planes), stride, 0, n, L, K, m.E, _lib.ptr(err), sh)
            _raise_invalid(trace, err, a)
        launch(planes, stride, 0, n, d_rel[i])
        free[j].record(comp)
    trace._validated = True
    comp.wait_stream(copy)


def trace_counts(trace: ActivationTrace):
    """Exact per-(layer, expert) selection counts as a device int64 [L, E] tensor (``mp_hist_u8``)."""
    t = _lib.torch()
    m = trace.model
    counts = t.zeros((m.L, m.E), dtype=t.int64, device=_lib.require_cuda())
    err = _lib.new_err()

    def launch(planes, stride, t0, t1, bounds):
        _lib.call("mp_hist_u8", _lib.ptr(planes), stride, t0, t1, m.L, m.K, m.E, _lib.ptr(counts), _lib.ptr(err),
                  _lib.stream_handle())

    sweep(trace, launch)
    _lib.check_err(err, "estimate_frequencies")
    return counts


def chunk_counts(trace: ActivationTrace):
    """Per-chunk load counts, device int64 [C, L, E] (``mp_hist_chunks_u8``): the sufficient
    statistics of every per-chunk hop sum (SPEC.md:383 linearity)."""
    t = _lib.torch()
    m = trace.model
    C = trace.n_chunks
    counts = t.zeros((C, m.L, m.E), dtype=t.int64, device=_lib.require_cuda())
    err = _lib.new_err()

    def launch(planes, stride, t0, t1, bounds):
        _lib.call("mp_hist_chunks_u8", _lib.ptr(planes), stride, t0, t1, m.L, m.K, m.E, _lib.ptr(bounds), C,
                  _lib.ptr(counts), _lib.ptr(err), _lib.stream_handle())

    sweep(trace, launch)
    _lib.check_err(err, "chunk_counts")
    return counts


def frequencies_from_counts(counts: np.ndarray, n_tokens: int, K: int) -> FrequencyTable:
    counts = np.asarray(counts, dtype=np.int64)
    return FrequencyTable(counts / (K * n_tokens), counts, int(n_tokens), int(K))


def estimate_frequencies(trace: ActivationTrace, model: Optional[ModelSpec] = None) -> FrequencyTable:
    """f[l, e] = count(l, e) / (K * n_tokens), counted on the GPU."""
    model = model or trace.model
    if trace.n_tokens == 0 or model is None:
        raise MoeplaceError("estimate_frequencies: empty trace (no silent uniform fallback)")
    if trace.model is not None and trace.model != model:
        raise ConfigError(f"trace shape {trace.model} does not match model {model}")
    counts = trace_counts(trace).cpu().numpy()
    return frequencies_from_counts(counts, trace.n_tokens, model.K)


def split_trace(trace: ActivationTrace, train_chunks: int, test_chunks: int):
    """the first ``train_chunks`` chunks (in id order) train, the next
    ``test_chunks`` test.  Both are zero-copy views of the same device planes."""
    if train_chunks < 0 or test_chunks < 0 or train_chunks + test_chunks > trace.n_chunks:
        raise ConfigError(f"cannot split {trace.n_chunks} chunks into {train_chunks} train + {test_chunks} test")
    return trace.view(0, train_chunks), trace.view(train_chunks, train_chunks + test_chunks)


def trace_stats(trace: ActivationTrace) -> dict:
    """Summary used by ``moeplace trace stats``."""
    freq = estimate_frequencies(trace)
    top = freq.f.max(axis=1)
    return {"n_tokens": trace.n_tokens, "n_chunks": trace.n_chunks,
            "L": trace.model.L, "E": trace.model.E, "K": trace.model.K,
            "max_f": float(top.max()), "mean_top1_f": float(top.mean()),
            "uniform_f": 1.0 / trace.model.E}
