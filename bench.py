#!/usr/bin/env python
"""Benchmark of the moeplace hot path on B200 (driver contract).

Workload (BASELINE.json configs[1], "config 2"): DeepSeek-R1 shape (L=58 MoE layers, E=256 experts,
top-K=8), 10M synthetic Zipf(s=1.2) tokens per GPU in 150 chunks per 10M tokens, FatTree
8 leaves x 4 servers x 8 GPUs (256 devices, 32 servers, 4 spines), c_layer=1, c_exp=64.
Placements scored: RR, Greedy, ILP and ILPLoad (P=4), computed in the untimed setup.

One step = one pass over the resident trace that builds the per-(layer, expert) load counts
(estimate_frequencies) AND scores the P=4 placements (per-chunk hop sums of evaluate), i.e.
"hist over all N and score of P=4 over all N" — by default with the fused kernel
(mp_hist_score_u8), or with --mode separate as mp_hist_u8 + mp_score_u8.  The library computes the
hop sums by count-contract (histogram of every (layer, chunk) piece contracted with the cost
tables at the piece's flush; exact by linearity); --algo gather times the per-byte
table gather instead (bit-identical results, tests/test_gpu_algos.py).  For N GPUs each rank
owns a contiguous 10M-token shard of one N*10M-token trace (weak scaling) and the packed int64
[counts | hop sums] buffer is combined with one NCCL all_reduce inside the timed step.

value  = token-layers scored x placements per second, whole job: N*10M*58*4 / step time.
e2e    = the same metric through the public API (moeplace.eval.evaluate_with_stats) on a trace
         held in pinned HOST memory: the H2D copy (streamed in slices, overlapped with the
         kernels), the kernels and the D2H of counts + sums are all inside the timed region.
--impl reference: the CPU restatement of the reference path (oracle/, numba, all host cores)
         on a bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

L, E, K = 58, 256, 8
ZIPF_S, SEED = 1.2, 0
TOK_PER_GPU = 10_000_000
CHUNKS_PER_GPU = 150
P = 4
METRIC = "token-layers scored/sec (x placements) and achieved HBM GB/s"
UNIT = "token-layers*placements/s"


def workload(n_gpus: int, tok: int, mode: str) -> dict:
    return {"workload": "config2: DeepSeek-R1 shape (L=58, E=256, K=8), Zipf(1.2) synthetic trace, "
                        f"{tok} tokens/GPU, {CHUNKS_PER_GPU} chunks/GPU, FatTree 8 leaves x 4 servers x 8 GPUs "
                        "(256 devices), c_layer=1, c_exp=64; per step: load histogram + hop sums of P=4 "
                        "placements (RR, Greedy, ILP, ILPLoad) over every token",
            "tokens_per_gpu": tok, "tokens_total": tok * n_gpus, "placements": P, "kernel_mode": mode,
            "l2": f"inputs larger than L2: {tok * L * K / 1e9:.2f} GB trace per GPU vs 126 MB L2, no flush needed",
            "parallelism": f"token shards x{n_gpus} + 1 NCCL all_reduce of int64 counts|sums" if n_gpus > 1
            else "single GPU"}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: an NVML polling thread
    (every ~2 ms), with `nvidia-smi -lms 100` as the fallback when NVML is unavailable."""

    # clocks_event_reasons bits (nvml.h): sw_power_cap 0x4, hw_slowdown 0x8, sw_thermal 0x20, hw_thermal 0x40
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.th = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self._stop.is_set():
                    self.sm.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for n, b in self.BITS.items():
                        if r & b:
                            self.reasons.add(n)
                    time.sleep(0.002)

            self.th = threading.Thread(target=poll, daemon=True)
            self.th.start()
        except Exception:
            self.th = None

    def stop(self) -> dict:
        self._stop.set()
        if self.th is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self.th.join(timeout=1)
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"], "samples": 0}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "sm_min_mhz": float(min(self.sm)), "source": "nvml",
                "window": "warm-up + timed steps (+ identical untimed steps until >= 8 samples)"}


def cpu_sample(trace, n_sample: int):
    """Token-major host copy of the first n_sample tokens of the device trace (same bytes)."""
    import torch
    v = trace.planes[:, trace.tok_begin * K:(trace.tok_begin + n_sample) * K].cpu().numpy()
    return np.ascontiguousarray(v.reshape(L, n_sample, K).transpose(1, 0, 2))


def time_oracle(sel, bounds, p, assigns, reps: int = 3, t0: int = 0):
    """Seconds per pass of the CPU restatement: counts + per-chunk hop sums of every placement
    in one token-block-parallel pass over the trace (oracle.evaluate.fused_pass)."""
    from oracle import evaluate as oe
    pes = [oe.pe_table(p, a) for a in assigns]
    oe.fused_pass(sel[:64], pes, bounds, E, t0)  # numba compile outside timing
    best = float("inf")
    for _ in range(reps):
        t_a = time.perf_counter()
        oe.fused_pass(sel, pes, bounds, E, t0)
        best = min(best, time.perf_counter() - t_a)
    return best


def host_info(run_1thread) -> dict:
    """SURVEY §8(d) CPU-baseline context: allowed CPUs, CPU model, NUMBA_NUM_THREADS and a
    single-thread rate (run_1thread() -> token-layers*placements/s with numba set to 1 thread)."""
    info = {"cpus_allowed": len(os.sched_getaffinity(0)),
            "numba_num_threads_env": os.environ.get("NUMBA_NUM_THREADS")}
    try:
        info["cpu_model"] = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name"))
    except Exception:  # noqa: BLE001
        pass
    try:
        import numba
        n0 = numba.get_num_threads()
        numba.set_num_threads(1)
        try:
            info["value_1thread"] = run_1thread()
        finally:
            numba.set_num_threads(n0)
    except Exception:  # noqa: BLE001
        pass
    return info


def cpu_threads() -> int:
    try:
        import numba
        return int(numba.get_num_threads())
    except Exception:
        return len(os.sched_getaffinity(0))


def run_reference(args, rank: int, world: int) -> None:
    """--impl reference: the reference path's CPU implementation (our oracle restatement of
    SPEC.md; the reference ships no code) on the host cores, bounded sample per step."""
    if rank != 0:
        return
    import numba
    from oracle import gen as og
    from oracle import topology as ot
    n_sample = args.ref_tokens
    sel, _ = og.generate(L, E, K, ZIPF_S, TOK_PER_GPU, CHUNKS_PER_GPU, SEED, tok_range=(0, n_sample))
    bounds = np.minimum(np.array([(c * TOK_PER_GPU + CHUNKS_PER_GPU - 1) // CHUNKS_PER_GPU
                                  for c in range(CHUNKS_PER_GPU + 1)]), n_sample)
    # FatTree 8x4x8 server graph: servers 0..31, leaves 32..39, spines 40..43
    links = [(s, 32 + s // 4) for s in range(32)] + [(32 + l, 40 + sp) for l in range(8) for sp in range(4)]
    dsrv = ot.server_hops(44, links, 32)
    dev_srv = np.repeat(np.arange(32), 8)
    disp = np.array([(l * 256) // L for l in range(L)])
    coll = np.concatenate([disp[1:], disp[-1:]])
    p = ot.cost_matrix(dsrv, dev_srv, disp, coll)
    rng = np.random.default_rng(0)
    assigns = [np.stack([rng.permutation(256) for _ in range(L)]).astype(np.int32) for _ in range(P)]
    threads = numba.get_num_threads()
    time_oracle(sel[:1000], bounds, p, assigns, reps=1)
    for _ in range(args.warmup):
        time_oracle(sel, bounds, p, assigns, reps=1)
    times = [time_oracle(sel, bounds, p, assigns, reps=1) for _ in range(args.steps)]
    t = float(np.mean(times))
    value = n_sample * L * P / t
    n1 = min(n_sample, 100_000)
    b1 = np.minimum(bounds, n1)
    host = host_info(lambda: n1 * L * P / time_oracle(sel[:n1], b1, p, assigns, reps=2))
    sample = (f"{n_sample} tokens (first {n_sample} of the config-2 trace, regenerated on the CPU), counts + "
              f"hop sums of {P} placements per step; numba parallel, {threads} threads")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": workload(world, TOK_PER_GPU, "cpu-oracle"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             **host, "sample_1thread": f"first {n1} tokens, 1 numba thread"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def bind_local_cpus(torch, local: int) -> None:
    """Restrict this rank to the CPUs local to its GPU (sysfs local_cpulist of the GPU's PCI
    function, intersected with the allowed set), so its pinned host buffers are first-touched on
    the GPU's NUMA node; a no-op on single-node hosts or when sysfs has no answer."""
    try:
        p = torch.cuda.get_device_properties(local)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        cl = open(f"/sys/bus/pci/devices/{bus}/local_cpulist").read().strip()
        cpus = set()
        for part in cl.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus and cpus != os.sched_getaffinity(0):
            os.sched_setaffinity(0, cpus)
    except Exception:  # noqa: BLE001 -- best effort
        pass


def emit(line):  # replaced in main() by a writer to the saved stdout descriptor
    print(json.dumps(line), flush=True)


def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", type=int, choices=[2, 3, 4, 5], default=2,
                    help="BASELINE config: 2 (default, the metric's config), 3 multi-topology, 4 4096 candidates, "
                         "5 100M tokens strong scaling")
    ap.add_argument("--mode", choices=["fused", "separate"], default="fused")
    ap.add_argument("--algo", choices=["auto", "gather", "count", "factorized"], default="auto",
                    help="hop-sum algorithm (include/moeplace_cuda.h MP_ALGO_*); auto = the library's choice "
                         "(config 4: factorized, as evaluate_many(method='auto') picks for P > 16)")
    ap.add_argument("--tokens", type=int, default=None, help="tokens per GPU (configs 2-4) / total (config 5)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-tokens", type=int, default=None, help="cpu_baseline sample (tokens)")
    ap.add_argument("--ref-tokens", type=int, default=1_000_000, help="--impl reference sample per step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # stdout carries exactly one JSON line: route library chatter (NCCL banner, warnings) to stderr
    sys.stdout.flush()
    json_fd = os.dup(1)
    os.dup2(2, 1)
    global emit
    emit = lambda line: os.write(json_fd, (json.dumps(line) + "\n").encode())  # noqa: E731
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import moeplace.eval as ev
    import moeplace.model_trace as mt
    import moeplace.placement as mpl
    import moeplace.solver as sv
    import moeplace.topology as topo
    from paper_2508_09229_b200 import _lib

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        bind_local_cpus(torch, local)  # pinned trace copies land on the GPU's NUMA node
        dist.init_process_group("nccl", device_id=dev)
    wl = args.workload
    model = mt.ModelSpec(L, E, K)
    c = mpl.Constraints(64, 1)

    def topology(kind, leaves, spl, gps, extra=None):
        g = topo.build_topology(topo.TopologySpec(kind, leaves, spl, gps, extra or {}))
        d = topo.all_pairs_hops(g)
        order = topo.locality_order(g, d)
        attn = mt.default_attention_placement(model, order)
        return g, d, order, attn, mpl.cost_matrix(d, attn)

    def methods(freq, g, order, attn, cost, which=("rr", "greedy", "ilp", "ilpload")):
        out = []
        for m in which:
            if m == "rr":
                pl = mpl.place_round_robin(model, attn, order, c)
            elif m == "greedy":
                pl = mpl.place_greedy(model, attn, cost, c)
            elif m == "ilp":
                pl = sv.solve_exact(sv.build_instance(cost, sv.UniformFrequencies(E), c))[0]
            else:
                pl = sv.solve_exact(sv.build_instance(cost, freq, c))[0]
            pl.label = f"{g.spec.kind}/{m}"
            out.append(pl)
        return out

    # ---------------- setup (untimed): trace shard, statistics, placements, tables ----------------
    if wl == 5:
        n_total = args.tokens or 100_000_000
        c_total = 1500
        a_tok, b_tok = (rank * n_total) // world, ((rank + 1) * n_total) // world
        scaling = "strong"
    else:
        per = args.tokens or (1_000_000 if wl == 4 else TOK_PER_GPU)
        n_total, c_total = per * world, CHUNKS_PER_GPU * world
        a_tok, b_tok = rank * per, (rank + 1) * per
        scaling = "weak"
    n = b_tok - a_tok
    trace = mt.generate_trace(model, ZIPF_S, n_total, c_total, SEED, tok_range=(a_tok, b_tok))
    counts0 = mt.trace_counts(trace)
    if world > 1:
        dist.all_reduce(counts0)
    freq = mt.frequencies_from_counts(counts0.cpu().numpy(), n_total, K)
    if wl in (2, 5):
        g, d, order, attn, cost = topology("FatTree", 8, 4, 8, {"spines": 4})
        placements = methods(freq, g, order, attn, cost)
        costs = [cost] * len(placements)
        kinds = ["FatTree 8x4x8"]
    elif wl == 3:
        placements, costs, kinds = [], [], []
        for kind in ("FatTree", "FatTreeHier", "Dragonfly", "DragonflySparse"):
            g, d, order, attn, cost = topology(kind, 16, 4, 4)
            pls = methods(freq, g, order, attn, cost)
            placements += pls
            costs += [cost] * len(pls)
            kinds.append(f"{kind} 16x4x4")
    else:
        g, d, order, attn, cost = topology("Dragonfly", 16, 4, 4)
        base = methods(freq, g, order, attn, cost, which=("ilpload",))[0]
        cand = mpl.perturb_swaps(base, 4096, 64, 1000)
        placements = [mpl.Placement(cand[i], c, f"cand{i}") for i in range(cand.shape[0])]
        costs = [cost] * len(placements)
        kinds = ["Dragonfly 16x4x4"]
    P_ = len(placements)
    C = trace.n_chunks
    planes, stride = trace.planes, trace.planes.shape[1]
    t0, t1 = trace.tok_begin, trace.tok_end
    bounds = _lib.to_dev(trace.chunk_bounds, torch.int64)
    err = _lib.new_err()
    stream = torch.cuda.current_stream()
    sh = _lib.stream_handle()
    fused = wl in (2, 5) and args.mode == "fused"
    groups = []  # (W, tables, max_p, n placements)
    if wl in (2, 5):
        tables, max_p = ev._group_tables(placements, costs, model, 1)
        groups.append((1, tables, max_p, P_))
    else:
        for g0 in range(0, P_, 16):
            grp = placements[g0:g0 + 16]
            W = ev._lanes_for(len(grp))
            tables, max_p = ev._group_tables(grp, costs[g0:g0 + 16], model, W)
            groups.append((W, tables, max_p, len(grp)))
    n_sums = sum(4 * W for W, _, _, _ in groups)
    with_hist = wl in (2, 5)
    buf = torch.zeros((L * E if with_hist else 0) + n_sums * C, dtype=torch.int64, device=dev)
    counts = buf[:L * E] if with_hist else None
    sums_all = buf[L * E:] if with_hist else buf
    views, off = [], 0
    for W, _, _, _ in groups:
        views.append(sums_all[off:off + 4 * W * C])
        off += 4 * W * C
    kev = [_events() for _ in range(2)]
    kernel_ms = [[], []]

    algo = {"auto": 0, "gather": 1, "count": 2, "factorized": 0}[args.algo]
    # config 4 (4096 candidates): the product path is evaluate_many(method="auto") -> factorized (one per-chunk
    # histogram pass + exact tensor-core contraction); the streaming passes are timed beside it
    fact = wl == 4 and args.algo in ("auto", "factorized")
    if args.algo == "factorized" and wl != 4:
        raise SystemExit("bench: --algo factorized applies to --workload 4")
    if fact:
        cnt_c4 = torch.zeros((C, L * E), dtype=torch.int64, device=dev)
        pe_all4 = ev.pe_matrix(placements, costs, model)
        out_f4 = torch.zeros((P_, C), dtype=torch.int64, device=dev)
        max_chunk = int(np.max(trace.chunk_token_counts()))
        max_pe4 = max(cs.max_p for cs in costs)
        kev_f = [_events() for _ in range(2)]

    def fstep(timed: bool):
        cnt_c4.zero_()
        if timed:
            kev_f[0][0].record(stream)
        _lib.call("mp_hist_chunks_u8", _lib.ptr(planes), stride, t0, t1, L, K, E, _lib.ptr(bounds), C,
                  _lib.ptr(cnt_c4), _lib.ptr(err), sh)
        if timed:
            kev_f[0][1].record(stream)
            kev_f[1][0].record(stream)
        out_f4.copy_(ev.contract_tc(cnt_c4, pe_all4, max_count=max_chunk, max_pe=max_pe4, err=err))
        if timed:
            kev_f[1][1].record(stream)
        if world > 1:
            dist.all_reduce(out_f4)

    def algo_used(hist: bool, W: int) -> str:  # mirrors choose_algo in csrc/stream.cu
        if args.algo not in ("auto", "factorized"):
            return {"gather": "gather", "count": "count-contract"}[args.algo]
        return "count-contract" if (hist or W > 1) else "gather"

    def step(timed: bool):
        buf.zero_()
        if with_hist and fused:
            if timed:
                kev[0][0].record(stream)
            W, tables, max_p, _ = groups[0]
            _lib.call("mp_hist_score_ex_u8", _lib.ptr(planes), stride, t0, t1, L, K, E, _lib.ptr(bounds), C,
                      _lib.ptr(tables), W, max_p, _lib.ptr(counts), _lib.ptr(views[0]), _lib.ptr(err), algo, sh)
            if timed:
                kev[0][1].record(stream)
        else:
            if with_hist:
                if timed:
                    kev[1][0].record(stream)
                _lib.call("mp_hist_u8", _lib.ptr(planes), stride, t0, t1, L, K, E, _lib.ptr(counts), _lib.ptr(err), sh)
                if timed:
                    kev[1][1].record(stream)
            if timed:
                kev[0][0].record(stream)
            for (W, tables, max_p, _), v in zip(groups, views):
                _lib.call("mp_score_ex_u8", _lib.ptr(planes), stride, t0, t1, L, K, _lib.ptr(bounds), C,
                          _lib.ptr(tables), W, max_p, _lib.ptr(v), algo, sh)
            if timed:
                kev[0][1].record(stream)
        if world > 1:
            dist.all_reduce(buf)

    # ---------------- CPU baseline (rank 0, N=1 only) ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        default_ns = {2: 1_000_000, 3: 250_000, 4: 2_000, 5: 1_000_000}[wl]
        ns = min(args.cpu_tokens or default_ns, n)
        sel = cpu_sample(trace, ns)
        bnd = np.minimum(np.asarray(trace.chunk_bounds, dtype=np.int64), ns)
        from oracle import evaluate as oe
        pes = []
        cache = {}
        for pl, cs in zip(placements, costs):
            key = id(cs)
            if key not in cache:
                cache[key] = cs.numpy()
            pes.append(oe.pe_table(cache[key], pl.assign))
        oe.fused_pass(sel[:16], pes, bnd, E)
        t_cpu = float("inf")
        for _ in range(5):
            t_a = time.perf_counter()
            oe.fused_pass(sel, pes, bnd, E)
            t_cpu = min(t_cpu, time.perf_counter() - t_a)
        thr = cpu_threads()
        cpu = {"value": ns * L * P_ / t_cpu, "unit": UNIT, "cores": thr, "kind": "port",
               "sample": f"first {ns} tokens of the same trace (D2H copy), counts + hop sums of the same {P_} "
                         f"placements in one pass, oracle/ numba parallel, best of 5, measured before any GPU timing",
               "ms_per_sample": t_cpu * 1e3}
        n1 = min(ns, 100_000 if wl != 4 else 500)
        b1 = np.minimum(bnd, n1)

        def one_thread():
            best = float("inf")
            for _ in range(2):
                t_a = time.perf_counter()
                oe.fused_pass(sel[:n1], pes, b1, E)
                best = min(best, time.perf_counter() - t_a)
            return n1 * L * P_ / best

        cpu.update(host_info(one_thread))
        cpu["sample_1thread"] = f"first {n1} tokens, 1 numba thread"

    launches_per_step = 1 if (fused or fact) else len(groups) + (1 if with_hist else 0)
    run = fstep if fact else step
    # the clock poller starts before the warm-up so it is already sampling when timing begins
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    for _ in range(args.warmup):
        run(False)
    torch.cuda.synchronize()
    if with_hist and not torch.equal(counts.view(L, E), counts0):
        raise SystemExit("bench: histogram of the timed pass differs from the setup histogram")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev_a, ev_b = _events()
    ev_a.record(stream)
    for _ in range(args.steps):
        run(False)
    ev_b.record(stream)
    torch.cuda.synchronize()
    for _ in range(args.steps):  # per-kernel shares with launch-bracketing events on the same stream
        run(True)
        torch.cuda.synchronize()
        ke = kev_f if fact else kev
        kernel_ms[0].append(ke[0][0].elapsed_time(ke[0][1]))
        if fact or (with_hist and not fused):
            kernel_ms[1].append(ke[1][0].elapsed_time(ke[1][1]))
    if world > 1:
        dist.barrier()
    if sampler and world == 1:
        # a short timed region can end before the poller has a handful of samples: keep the GPU on
        # the identical (untimed) step until it has >= 8, so the reported clocks are under this load
        extra = 0
        while len(sampler.sm) < 8 and extra < 2000:
            run(False)
            extra += 1
            if extra % 50 == 0:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    _lib.check_err(err, "bench: device data error in the timed steps")
    t_step = torch.tensor([ev_a.elapsed_time(ev_b) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_step, op=dist.ReduceOp.MAX)
    ms = float(t_step.item())
    value = n_total * L * P_ / (ms / 1e3)

    # ---------------- roofline of the dominant kernel ----------------
    peak, peak_src = measured_peak()
    k_main = float(np.mean(kernel_ms[0]))
    if fused:
        kname, tkey, launches = ("mp_hist_score_u8 (fused hist+score of 4 placements; count-contract: histogram "
                                 "+ per-(layer,chunk) contraction with the cost tables)"), "fused", 1
    elif fact:
        kname, tkey, launches = ("mp_hist_chunks_u8 (factorized evaluator: per-chunk histogram int64 [C][L][E]; "
                                 "the exact contraction with the 4096 pe rows runs after it as cuBLASLt int8 GEMMs)"), \
            "hist_chunks", 1
    else:
        Ws = sorted({W for W, _, _, _ in groups})
        kname = f"mp_score_u8 (W={'/'.join(map(str, Ws))}, {len(groups)} launch(es) per step)"
        tkey, launches = ("score" if Ws == [1] else f"score_w{Ws[-1]}"), len(groups)
        if with_hist and np.mean(kernel_ms[1]) > k_main:
            k_main, kname, tkey, launches = float(np.mean(kernel_ms[1])), "mp_hist_u8", "hist", 1
    alg_bytes = n * L * K  # one u8 id per (token, layer, pick), per launch
    per_launch_ms = k_main / launches
    achieved = alg_bytes / (per_launch_ms / 1e3) / 1e9
    traffic = None
    try:
        tr = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        ent = tr.get(tkey, {})
        if ent.get("tokens"):
            traffic = ent["dram_bytes_per_launch"] * n / ent["tokens"]  # scaled to this launch's tokens
    except Exception:
        traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kname, "kernel_ms_per_launch": per_launch_ms,
                "kernel_share_of_step": k_main / ms if world == 1 else None, "alg_bytes_per_launch": alg_bytes,
                "peak_source": peak_src}
    if with_hist and not fused:
        roofline["hist_ms"] = float(np.mean(kernel_ms[1]))
    if fact:
        roofline["contraction_ms"] = float(np.mean(kernel_ms[1]))
    if wl in (3, 4) and not fact and algo_used(False, 4) == "gather":
        # shared-memory roofline for the W=4 gather: 4 LDS.128 wavefronts per 32 lookups + 4 LDG wavefronts
        # per 512 B, at 1 wavefront / SM / clock (sm_max_mhz)
        mhz = (clocks or {}).get("sm_mhz") or 1965.0
        lookups = n * L * K
        wf = lookups / 32 * 4 * 4 / 4 + n * L * K / 512 * 4  # per launch group of 16 placements
        roofline["smem_bound_ms_per_launch"] = wf / 148 / (mhz * 1e6) * 1e3

    # ---------------- each streaming kernel alone on the same trace (context for the roofline) ----------
    kernels_alone = None
    if wl in (2, 5) and rank == 0:
        scratch = torch.zeros_like(buf)
        alone = {
            "mp_score_u8 (W=1, 4 placements)": lambda: _lib.call(
                "mp_score_u8", _lib.ptr(planes), stride, t0, t1, L, K, _lib.ptr(bounds), C,
                _lib.ptr(groups[0][1]), 1, groups[0][2], _lib.ptr(scratch[L * E:]), sh),
            "mp_hist_u8": lambda: _lib.call(
                "mp_hist_u8", _lib.ptr(planes), stride, t0, t1, L, K, E, _lib.ptr(scratch[:L * E]), _lib.ptr(err), sh),
            # the same fused step with the per-byte GATHER algorithm (one LDS per lookup + ATOMS), for comparison
            "mp_hist_score_ex_u8 (GATHER, 4 placements)": lambda: _lib.call(
                "mp_hist_score_ex_u8", _lib.ptr(planes), stride, t0, t1, L, K, E, _lib.ptr(bounds), C,
                _lib.ptr(groups[0][1]), 1, groups[0][2], _lib.ptr(scratch[:L * E]), _lib.ptr(scratch[L * E:]),
                _lib.ptr(err), 1, sh),
        }
        kernels_alone = {}
        for nm, fn in alone.items():
            for _ in range(3):
                fn()
            xa, xb = _events()
            xa.record(stream)
            for _ in range(10):
                fn()
            xb.record(stream)
            torch.cuda.synchronize()
            kms_ = xa.elapsed_time(xb) / 10
            gbs = n * L * K / (kms_ / 1e3) / 1e9
            kernels_alone[nm] = {"ms": kms_, "GBps": gbs, "frac": gbs / peak}
        # L1TEX model (the SM's L1TEX/shared pipe moves one wavefront per clock): the step's wavefronts per
        # launch are the shared-memory wavefronts ncu counted for the same kernel on the same trace
        # (profiles/traffic.json, from the committed --set full capture; ATOMS + flush reads) plus one per
        # 128 B of coalesced LDG.128; bound = wavefronts / (148 SMs x SM clock).
        mhz = (clocks or {}).get("sm_mhz") or 1965.0
        clk = mhz * 1e6
        if fused:
            try:
                ent = json.loads((ROOT / "profiles" / "traffic.json").read_text())["fused"]
                shw = ent["shared_wavefronts_per_launch"] * n / ent["tokens"]
            except Exception:
                shw = None
            if shw:
                ldg = n * L * K / 128
                bound = (shw + ldg) / 148 / clk * 1e3
                roofline["l1tex_model"] = {
                    "shared_wavefronts_per_launch": shw, "ldg_wavefronts_per_launch": ldg,
                    "wavefronts_per_512B": (shw + ldg) / (n * L * K / 512), "sm_mhz": mhz, "bound_ms": bound,
                    "frac_of_l1tex_bound": bound / per_launch_ms,
                    "shared_wavefronts_per_atoms_instr": shw / (n * L * K / 32),
                    "source": "ncu --set full capture (profiles/r1_ncu_summary.md): "
                              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"}

    # ------- configs 2/4: the factorized evaluator beside the measured gather (not the headline) -------
    factorized = None
    passes = None
    if fact:
        # the same 4096 hop sums by 256 streaming passes of 16 placements (count-contract), for comparison
        for _ in range(2):
            step(False)
        torch.cuda.synchronize()
        ok = torch.equal(out_f4, sums_all[:P_ * C].view(P_, C))
        pa, pb = _events()
        n_p = max(3, args.steps // 4)
        pa.record(stream)
        for _ in range(n_p):
            step(False)
        pb.record(stream)
        torch.cuda.synchronize()
        p_ms = pa.elapsed_time(pb) / n_p
        passes = {"ms_per_step": p_ms, "launches_per_step": len(groups), "algorithm": algo_used(False, 4),
                  "value": n_total * L * P_ / (p_ms / 1e3), "bit_identical_to_step": ok,
                  "hbm_frac_per_pass": n * L * K / (p_ms / len(groups) / 1e3) / 1e9 / peak,
                  "note": "evaluate_many(method='count'): 256 mp_score_u8 W=4 passes over the resident trace"}
    if wl == 2 or (wl == 4 and not fact):
        cnt_c = torch.zeros((C, L * E), dtype=torch.int64, device=dev)
        pe_all = ev.pe_matrix(placements, costs, model)
        out_f = torch.zeros((P_, C), dtype=torch.int64, device=dev)

        def fstep():
            cnt_c.zero_()
            _lib.call("mp_hist_chunks_u8", _lib.ptr(planes), stride, t0, t1, L, K, E, _lib.ptr(bounds), C,
                      _lib.ptr(cnt_c), _lib.ptr(err), sh)
            out_f.copy_(ev.contract_tc(cnt_c, pe_all))
            if with_hist:
                torch.sum(cnt_c, 0, out=cnt_tot)  # the load histogram is the sum of the per-chunk ones

        cnt_tot = torch.zeros(L * E, dtype=torch.int64, device=dev)
        for _ in range(3):
            fstep()
        torch.cuda.synchronize()
        ok = torch.equal(out_f, sums_all[:P_ * C].view(P_, C)) if world == 1 else None
        if ok and with_hist:
            ok = torch.equal(cnt_tot.view(L, E), counts0)
        fa, fb = _events()
        fa.record(stream)
        for _ in range(args.steps):
            fstep()
        fb.record(stream)
        torch.cuda.synchronize()
        f_ms = fa.elapsed_time(fb) / args.steps
        factorized = {"ms_per_step": f_ms, "placements_evaluated_per_s": P_ / (f_ms / 1e3),
                      "bit_identical_to_step": ok,
                      "note": "cross-check: per-chunk histogram materialised in HBM (mp_hist_chunks_u8, int64 [C][L][E]) "
                              "+ exact contraction on the tensor cores (7-bit digit int8 GEMMs, cuBLASLt, int32 "
                              "accumulation) -- the out-of-kernel form of the step's count-contract; "
                              "same per-chunk hop sums by linearity (SPEC.md:383)"}

    # ---------------- e2e through the public API, host buffers ----------------
    e2e = None
    if not args.no_e2e:
        host = trace.to_host(pin=True)
        cand_host = torch.from_numpy(cand).pin_memory() if fact else None
        steps_e = max(1, args.e2e_steps if wl != 5 else 1)

        def api_call():
            if with_hist:
                return ev.evaluate_with_stats(host, placements, costs[0])[0].counts
            if fact:  # the candidate batch as one pinned host array, as a search loop holds it
                return ev.evaluate_batch(host, cand_host, costs[0])  # auto -> factorized for P > 16
            return ev.score_sums(host, placements, costs)

        api_call()  # warm-up
        evs = []
        for _ in range(steps_e):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            a, b = _events()
            a.record(stream)
            res = api_call()  # H2D (streamed, overlapped) + kernels + D2H + host floats
            b.record(stream)
            torch.cuda.synchronize()
            evs.append(a.elapsed_time(b))
        if with_hist and world == 1 and not np.array_equal(res, counts0.cpu().numpy()):
            raise SystemExit("bench: e2e histogram differs")
        t_e = torch.tensor([float(np.mean(evs))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        e_ms = float(t_e.item())
        api = ("moeplace.eval.evaluate_with_stats(trace in pinned host memory, 4 placements, cost)" if with_hist
               else f"moeplace.eval.evaluate_batch(trace and the int32 [{P_}, L, E] candidate batch in pinned host "
                    f"memory, method='auto' -> factorized; pe tables, contraction and per-candidate floats inside "
                    f"the call)" if fact
               else f"moeplace.eval.score_sums(trace in pinned host memory, {P_} placements)")
        e2e = {"value": n_total * L * P_ / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(n * L * K * world + (cand.nbytes if fact else 0)),
               "d2h_bytes_per_step": int(((L * E if with_hist else 0) + P_ * C) * 8 * world), "api": api}
        del host

    if rank == 0:
        cfg = workload(world, n, "fused" if fused else "separate")
        if wl != 2:
            cfg = {"workload": {3: "config3: DeepSeek-R1 shape, 10M Zipf(1.2) tokens/GPU, 16 placements (RR, Greedy, "
                                   "ILP, ILPLoad) x 4 topologies (FatTree, FatTreeHier, Dragonfly, DragonflySparse, "
                                   "16x4x4 = 256 devices) scored in one W=4 pass",
                                4: "config4: DeepSeek-R1 shape, 1M Zipf(1.2) tokens/GPU, Dragonfly 16x4x4, 4096 candidate "
                                   "placements (ILPLoad + 64 within-layer swaps each, seeds 1000+i) scored per step "
                                   + ("(factorized: one per-chunk histogram pass + exact int8 tensor-core contraction, "
                                      "what evaluate_many(method='auto') runs for P > 16)" if fact
                                      else "(256 W=4 passes)"),
                                5: f"config5: DeepSeek-R1 shape, {n_total} Zipf(1.2) tokens total sharded over "
                                   f"{world} GPU(s), 1500 chunks, FatTree 8x4x8; hist + score of 4 placements"}[wl],
                   "tokens_per_gpu": n, "tokens_total": n_total, "placements": P_, "topologies": kinds,
                   "l2": f"inputs larger than L2 ({n * L * K / 1e9:.2f} GB/GPU vs 126 MB)" if n * L * K > 126e6
                   else f"trace {n * L * K / 1e6:.0f} MB < 126 MB L2: each step streams it {len(groups)}x; "
                        "first pass per step from HBM, reuse from L2",
                   "parallelism": f"token shards x{world}" + (" + 1 NCCL all_reduce" if world > 1 else "")}
        cfg["hop_sum_algorithm"] = (algo_used(True, 1) if fused else "factorized" if fact else
                                    "/".join(sorted({algo_used(False, W) for W, _, _, _ in groups})))
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "u8", "data": "synthetic (counter-based Zipf generator, seed 0)",
                "config": cfg, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches_per_step * args.steps, "clocks": clocks, "factorized": factorized,
                "passes": passes,
                "kernels_alone": kernels_alone,
                "hbm_gbs_step": n * L * K / (ms / 1e3) / 1e9}
        emit(line)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
