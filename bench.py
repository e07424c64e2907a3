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
[counts | hop sums] buffer is summed inside the timed step by the library's NVLink/NVSwitch peer-memory kernel
(symmetric memory, multimem.ld_reduce; `--collective nccl` uses one NCCL all_reduce instead).

value  = token-layers scored x placements per second, whole job: N*10M*58*4 / step time.
e2e    = the same metric through the public API (moeplace.eval.evaluate_with_stats) on the SPEC's
         token-major [N, L, K] selections held in pinned HOST memory: the H2D copy (streamed in
         slices, overlapped with the kernels), the on-device transpose into layer planes, the
         kernels and the D2H of counts + sums are all inside the timed region.
--impl reference: the CPU restatement of the reference path (oracle/, numba, all host cores) on
         the same trace (regenerated on the CPU by the oracle's sampler), the same placements and
         the same topology (bench_data/placements_wl*.npz, written by this script's GPU arm with
         --write-fixtures and checked by it on every run); rank 0 only.
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
METRIC = "token-layers scored/sec (x placements) and achieved HBM GB/s"
UNIT = "token-layers*placements/s"
FIXTURES = ROOT / "bench_data"
CPU_BLOCK = 1_000_000  # the CPU legs stream the trace in 1M-token blocks
CONFIG3_KINDS = (("FatTree", 16), ("FatTreeHier", 16), ("Dragonfly", 16), ("DragonflySparse", 16),
                 ("DragonflyPlus", 16), ("SlimFly", 18))


def shape_of(wl: int, n_gpus: int, tokens_arg):
    """(tokens per GPU, total tokens, total chunks, scaling) of a workload."""
    if wl == 5:
        n_total = tokens_arg or 100_000_000
        return n_total // n_gpus, n_total, 1500, "strong"
    per = tokens_arg or (1_000_000 if wl == 4 else TOK_PER_GPU)
    return per, per * n_gpus, CHUNKS_PER_GPU * n_gpus, "weak"


def workload(wl: int, n_gpus: int, tok: int, n_total: int, P: int) -> dict:
    """The `config` object: identical for the GPU arm and the reference arm (same workload)."""
    desc = {
        2: "config2: DeepSeek-R1 shape (L=58, E=256, K=8), Zipf(1.2) synthetic trace, "
           f"{tok} tokens/GPU, {CHUNKS_PER_GPU} chunks/GPU, FatTree 8 leaves x 4 servers x 8 GPUs "
           "(256 devices), c_layer=1, c_exp=64; per step: load histogram + hop sums of P=4 "
           "placements (RR, Greedy, ILP, ILPLoad) over every token",
        3: f"config3: DeepSeek-R1 shape, {tok} Zipf(1.2) tokens/GPU, {CHUNKS_PER_GPU} chunks, 24 placements (RR, "
           "Greedy, ILP, ILPLoad) x 6 topologies (FatTree, FatTreeHier, Dragonfly, DragonflySparse, DragonflyPlus "
           "16x4x4 = 256 devices; SlimFly 18x4x4 = 288 devices), c_layer=1, c_exp=64; per step: hop sums of all 24",
        4: f"config4: DeepSeek-R1 shape, {tok} Zipf(1.2) tokens/GPU, Dragonfly 16x4x4, 4096 candidate placements "
           "(ILPLoad + 64 within-layer swaps each, seeds 1000+i); per step: per-chunk hop sums of all 4096",
        5: f"config5: DeepSeek-R1 shape, {n_total} Zipf(1.2) tokens total sharded over {n_gpus} GPU(s), 1500 chunks, "
           "FatTree 8x4x8; per step: load histogram + hop sums of P=4 placements (RR, Greedy, ILP, ILPLoad)",
    }[wl]
    by = tok * L * K
    return {"workload": desc, "tokens_per_gpu": tok, "tokens_total": n_total, "placements": P,
            "l2": (f"inputs larger than L2: {by / 1e9:.2f} GB trace per GPU vs 126 MB L2, no flush needed" if by > 126e6
                   else f"trace {by / 1e6:.0f} MB < 126 MB L2 (reused across the step's passes)"),
            "parallelism": (f"token shards x{n_gpus} + 1 sum of the int64 counts|sums vector over NVLink/NVSwitch "
                            "peer memory (library kernel, multimem.ld_reduce; NCCL all_reduce with --collective nccl)"
                            if n_gpus > 1
                            else "single GPU")}


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
        return self

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


# ------------------------------ CPU legs (oracle; test infrastructure) ------------------------------

def load_fixture(wl: int):
    """Placements and cost matrices the GPU arm scores (written by `bench.py --write-fixtures`):
    (labels, [assign int32 [L, E]], [p uint8 [L, S]] per placement)."""
    key = {2: 2, 5: 2, 3: 3, 4: 4}[wl]
    path = FIXTURES / f"placements_wl{key}.npz"
    d = np.load(path)
    labels = [str(x) for x in d["labels"]]
    assigns = [d["assign"][i].astype(np.int32) for i in range(len(labels))]
    costs = [d[f"p{int(t)}"] for t in d["topo_of"]]
    return labels, assigns, costs, str(path.relative_to(ROOT))


def perturb_swaps_np(base: np.ndarray, n: int, n_swaps: int, seed0: int) -> np.ndarray:
    """Config-4 candidates, restated for the CPU leg (placement.perturb_swaps):
    candidate i = `n_swaps` within-layer swaps of `base` drawn with seed seed0 + i."""
    Lb, Eb = base.shape
    out = np.repeat(base[None], n, axis=0).astype(np.int32)
    for i in range(n):
        rng = np.random.default_rng(seed0 + i)
        ls, a, b = rng.integers(0, Lb, n_swaps), rng.integers(0, Eb, n_swaps), rng.integers(0, Eb, n_swaps)
        c = out[i]
        for l, x, y in zip(ls, a, b):
            c[l, x], c[l, y] = c[l, y], c[l, x]
    return out


def cpu_setup(wl: int, n_tokens: int, n_chunks: int, a_tok: int, n_sample: int):
    """The CPU legs' inputs: the oracle regenerates tokens [a_tok, a_tok + n_sample) of the SAME
    trace in 1M-token blocks (parallel first touch, like any numba-parallel producer), and the
    placements / cost matrices come from the committed fixture.  Returns (blocks [(t0, sel)],
    bounds, pes, labels, fixture path)."""
    from oracle import evaluate as oe
    from oracle import gen as og
    labels, assigns, costs, fx = load_fixture(wl)
    if wl == 4:
        base = assigns[0]
        assigns = list(perturb_swaps_np(base, 4096, 64, 1000))
        costs = costs * len(assigns)
        labels = [f"cand{i}" for i in range(len(assigns))]
    pes = [oe.pe_table(p, a) for p, a in zip(costs, assigns)]
    blocks = []
    for s0 in range(a_tok, a_tok + n_sample, CPU_BLOCK):
        s1 = min(s0 + CPU_BLOCK, a_tok + n_sample)
        sel, bounds = og.generate(L, E, K, ZIPF_S, n_tokens, n_chunks, SEED, tok_range=(s0, s1))
        blocks.append((s0, sel))
    bounds = np.array([(c * n_tokens + n_chunks - 1) // n_chunks for c in range(n_chunks + 1)], dtype=np.int64)
    return blocks, bounds, pes, labels, fx


def cpu_pass(blocks, pes, bounds):
    """One pass of the CPU restatement over the blocks: load counts [L, E] and per-chunk hop sums
    [P, C] (oracle.evaluate.fused_pass: token blocks on all numba threads, private partials,
    integer merge), summed over the blocks."""
    from oracle import evaluate as oe
    cnt, sums = None, None
    for t0, sel in blocks:
        c, s = oe.fused_pass(sel, pes, bounds, E, t0)
        cnt = c if cnt is None else cnt + c
        sums = s if sums is None else sums + s
    return cnt, sums


def time_cpu(blocks, pes, bounds, steps: int, warmup: int):
    from oracle import evaluate as oe
    oe.fused_pass(blocks[0][1][:64], pes, bounds, E, blocks[0][0])  # numba compile outside timing
    for _ in range(warmup):
        cpu_pass(blocks, pes, bounds)
    ts = []
    for _ in range(steps):
        t_a = time.perf_counter()
        res = cpu_pass(blocks, pes, bounds)
        ts.append(time.perf_counter() - t_a)
    return float(np.mean(ts)), res


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


def cpu_leg(wl, n_total, c_total, a_tok, n_sample, steps, warmup):
    """Shared by the reference arm and the GPU arm's cpu_baseline: the same code, input and
    timing rule (mean over `steps` passes after `warmup`), so the two CPU numbers agree."""
    blocks, bounds, pes, labels, fx = cpu_setup(wl, n_total, c_total, a_tok, n_sample)
    t, res = time_cpu(blocks, pes, bounds, steps, warmup)
    P = len(pes)
    n1 = min(n_sample, 100_000 if wl != 4 else 500)
    b1 = [(blocks[0][0], blocks[0][1][:n1])]

    def one_thread():
        t1, _ = time_cpu(b1, pes, bounds, 1, 0)
        return n1 * L * P / t1

    info = host_info(one_thread)
    thr = cpu_threads()
    d = {"value": n_sample * L * P / t, "unit": UNIT, "cores": thr, "kind": "port",
         "sample": (f"tokens [{a_tok}, {a_tok + n_sample}) of the workload's trace, regenerated on the CPU by the "
                    f"oracle sampler in {len(blocks)} block(s) of <= {CPU_BLOCK} tokens; counts + per-chunk hop sums "
                    f"of the same {P} placements (fixture {fx}) in one oracle pass per block, numba parallel, "
                    f"{thr} threads; mean of {steps} passes after {warmup} warm-up"),
         "ms_per_pass": t * 1e3, **info, "sample_1thread": f"first {n1} tokens, 1 numba thread"}
    return d, res, labels, bounds


def run_reference(args, rank: int, world: int) -> None:
    """--impl reference: the reference path's CPU implementation (our oracle restatement of
    SPEC.md; the reference ships no code) on the host cores: the same trace (regenerated by the
    oracle sampler), placements and topology as the GPU arm; configs 2 and 3 time all 10M tokens
    streamed in 1M-token blocks, configs 4 and 5 a bounded sample."""
    if rank != 0:
        return
    wl = args.workload
    tok, n_total, c_total, scaling = shape_of(wl, world, args.tokens)
    default = {2: tok, 3: tok, 4: 5_000, 5: 10_000_000}[wl]
    n_sample = min(args.ref_tokens or default, tok if wl != 5 else n_total)
    cb, _, labels, _ = cpu_leg(wl, n_total, c_total, 0, n_sample, args.steps, args.warmup)
    P = len(labels)
    value = cb["value"]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_pass"], "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "u8", "data": "synthetic (counter-based Zipf generator, seed 0)",
            "config": workload(wl, world, tok, n_total, P), "cpu_baseline": cb,
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
                    help="BASELINE config: 2 (default, the metric's config), 3 six topologies x 4 methods, 4 4096 "
                         "candidates, 5 100M tokens strong scaling")
    ap.add_argument("--mode", choices=["fused", "separate"], default="fused")
    ap.add_argument("--algo", choices=["auto", "gather", "count", "seg", "token", "factorized"], default="auto",
                    help="hop-sum algorithm (include/moeplace_cuda.h MP_ALGO_*); auto = the library's choice "
                         "(config 4: factorized, as evaluate_many(method='auto') picks for P > 16)")
    ap.add_argument("--tokens", type=int, default=None, help="tokens per GPU (configs 2-4) / total (config 5)")
    ap.add_argument("--chunks", type=int, default=None,
                    help="chunks per GPU (default 150; e.g. 71429 = ~140 tokens per chunk, the paper's dialog length)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-tokens", type=int, default=None, help="cpu_baseline sample (tokens)")
    ap.add_argument("--ref-tokens", type=int, default=None, help="--impl reference sample per step")
    ap.add_argument("--sustained-s", type=float, default=0.6, help="seconds of back-to-back steps for the sustained figure")
    ap.add_argument("--write-fixtures", default=None, help="directory: save the placements the CPU legs use")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--collective", choices=["peer", "nccl"], default="peer",
                    help="N > 1: sum the packed result with the library's NVLink/NVSwitch peer-memory kernel "
                         "(default) or with torch.distributed.all_reduce (NCCL)")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    global CHUNKS_PER_GPU
    if args.chunks:
        CHUNKS_PER_GPU = args.chunks

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
    from paper_2508_09229_b200.shard import PeerSum

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
    n, n_total, c_total, scaling = shape_of(wl, world, args.tokens)
    a_tok, b_tok = rank * n, (rank + 1) * n
    if wl == 5:
        a_tok, b_tok = (rank * n_total) // world, ((rank + 1) * n_total) // world
        n = b_tok - a_tok
    else:
        c_total = CHUNKS_PER_GPU * world
    trace = mt.generate_trace(model, ZIPF_S, n_total, c_total, SEED, tok_range=(a_tok, b_tok))
    counts0 = mt.trace_counts(trace)
    if world > 1:
        dist.all_reduce(counts0)
    freq = mt.frequencies_from_counts(counts0.cpu().numpy(), n_total, K)
    topo_costs = []  # distinct cost matrices, in fixture order
    if wl in (2, 5):
        g, d, order, attn, cost = topology("FatTree", 8, 4, 8, {"spines": 4})
        placements = methods(freq, g, order, attn, cost)
        costs = [cost] * len(placements)
        kinds = ["FatTree 8x4x8"]
        topo_costs = [cost]
    elif wl == 3:
        placements, costs, kinds = [], [], []
        for kind, leaves in CONFIG3_KINDS:
            g, d, order, attn, cost = topology(kind, leaves, 4, 4)
            pls = methods(freq, g, order, attn, cost)
            placements += pls
            costs += [cost] * len(pls)
            kinds.append(f"{kind} {leaves}x4x4")
            topo_costs.append(cost)
    else:
        g, d, order, attn, cost = topology("Dragonfly", 16, 4, 4)
        base = methods(freq, g, order, attn, cost, which=("ilpload",))[0]
        cand = mpl.perturb_swaps(base, 4096, 64, 1000)
        placements = [mpl.Placement(cand[i], c, f"cand{i}") for i in range(cand.shape[0])]
        costs = [cost] * len(placements)
        kinds = ["Dragonfly 16x4x4"]
        topo_costs = [cost]
    P_ = len(placements)

    # the CPU legs score the same placements: save / check the committed fixture
    fx_src = [base] if wl == 4 else placements
    fx_topo = [0] if wl == 4 else [next(i for i, u in enumerate(topo_costs) if u is cs) for cs in costs]
    fx = {"labels": np.array([p.label or "" for p in fx_src]),
          "assign": np.stack([p.assign for p in fx_src]).astype(np.int16), "topo_of": np.array(fx_topo, np.int32)}
    for i, cs in enumerate(topo_costs):
        fx[f"p{i}"] = cs.numpy().astype(np.uint8)
    fx_key = {2: 2, 5: 2, 3: 3, 4: 4}[wl]
    if args.write_fixtures and rank == 0 and not (wl == 5 or args.tokens or args.chunks):
        os.makedirs(args.write_fixtures, exist_ok=True)
        np.savez_compressed(Path(args.write_fixtures) / f"placements_wl{fx_key}.npz", **fx)
    fixture_match = None
    try:
        ref = np.load(FIXTURES / f"placements_wl{fx_key}.npz")
        fixture_match = bool(all(np.array_equal(ref[k], fx[k]) for k in fx if k != "labels"))
    except Exception:  # noqa: BLE001
        fixture_match = None

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
        lanes = ev.pass_lanes(trace, costs)  # 32 per count-contract pass (config 3: P = 24 in one pass)
        for g0 in range(0, P_, lanes):
            grp = placements[g0:g0 + lanes]
            W = ev._lanes_for(len(grp))
            tables, max_p = ev._group_tables(grp, costs[g0:g0 + lanes], model, W)
            groups.append((W, tables, max_p, len(grp)))
    n_sums = sum(4 * W for W, _, _, _ in groups)
    with_hist = wl in (2, 5)
    # N > 1: the packed [counts | sums] vector lives in symmetric memory and is summed over NVLink /
    # NVSwitch by the library's own kernel (shard.PeerSum, multimem.ld_reduce); --collective nccl
    # uses torch.distributed.all_reduce instead
    n_buf = (L * E if with_hist else 0) + n_sums * C
    peer = PeerSum.create(n_buf) if world > 1 and args.collective == "peer" else None
    buf = torch.zeros(n_buf, dtype=torch.int64, device=dev)

    def carve(b):
        """[counts | sums] views of one packed buffer: (counts or None, [sums view per group])."""
        sums_all = b[L * E:] if with_hist else b
        vs, off = [], 0
        for W, _, _, _ in groups:
            vs.append(sums_all[off:off + 4 * W * C])
            off += 4 * W * C
        return (b[:L * E] if with_hist else None), vs

    counts, views = carve(buf)  # the step's result (after the cross-GPU sum when N > 1)

    algo = {"auto": 0, "gather": 1, "count": 2, "token": 3, "seg": 4, "factorized": 0}[args.algo]
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

    def fstep(hi=None):
        cnt_c4.zero_()
        _lib.call("mp_hist_chunks_u8", _lib.ptr(planes), stride, t0, hi or t1, L, K, E, _lib.ptr(bounds), C,
                  _lib.ptr(cnt_c4), _lib.ptr(err), sh)
        out_f4.zero_()
        ev.CountDigits(cnt_c4, max_chunk, err).contract(pe_all4, out_f4)  # 8-bit count digits + tcgen05 kind::i8 GEMM
        if world > 1:
            dist.all_reduce(out_f4)

    def step(hi=None):
        nonlocal counts, views
        hi = hi or t1
        b = peer.input() if peer is not None else buf  # peer: this epoch's half of the symmetric pair
        b.zero_()
        cnt_b, views_b = carve(b)
        if with_hist and fused:
            W, tables, max_p, _ = groups[0]
            _lib.call("mp_hist_score_ex_u8", _lib.ptr(planes), stride, t0, hi, L, K, E, _lib.ptr(bounds), C,
                      _lib.ptr(tables), W, max_p, _lib.ptr(cnt_b), _lib.ptr(views_b[0]), _lib.ptr(err), algo, sh)
        else:
            if with_hist:
                _lib.call("mp_hist_u8", _lib.ptr(planes), stride, t0, hi, L, K, E, _lib.ptr(cnt_b), _lib.ptr(err), sh)
            for (W, tables, max_p, _), v in zip(groups, views_b):
                _lib.call("mp_score_ex_u8", _lib.ptr(planes), stride, t0, hi, L, K, _lib.ptr(bounds), C,
                          _lib.ptr(tables), W, max_p, _lib.ptr(v), algo, sh)
        if peer is not None:
            counts, views = carve(peer.allreduce())
        elif world > 1:
            dist.all_reduce(b)

    def main_kernel():
        """The step's dominant kernel alone (no zeroing, no collective): the roofline numerator."""
        if fact:
            _lib.call("mp_hist_chunks_u8", _lib.ptr(planes), stride, t0, t1, L, K, E, _lib.ptr(bounds), C,
                      _lib.ptr(cnt_c4), _lib.ptr(err), sh)
        elif fused:
            W, tables, max_p, _ = groups[0]
            _lib.call("mp_hist_score_ex_u8", _lib.ptr(planes), stride, t0, t1, L, K, E, _lib.ptr(bounds), C,
                      _lib.ptr(tables), W, max_p, _lib.ptr(counts), _lib.ptr(views[0]), _lib.ptr(err), algo, sh)
        else:
            W, tables, max_p, _ = groups[0]
            _lib.call("mp_score_ex_u8", _lib.ptr(planes), stride, t0, t1, L, K, _lib.ptr(bounds), C,
                      _lib.ptr(tables), W, max_p, _lib.ptr(views[0]), algo, sh)

    def algo_used(hist: bool, W: int) -> str:
        if fact:
            return "factorized"
        if args.algo != "auto":
            return {"gather": "gather", "count": "count-contract", "seg": "segmented gather",
                    "token": "token-tiled"}[args.algo]
        mp_ = max(g[2] for g in groups)
        a = _lib.choose_algo(hist, W, n, C, L, K, mp_)  # the library's own AUTO rule
        return {"gather": "gather", "count": "count-contract", "token": "token-tiled", "seg": "segmented gather"}[a]

    run = fstep if fact else step

    # ---------------- CPU baseline + parity sample (rank 0, N=1 only; before any GPU timing) ----------------
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        default_ns = {2: 1_000_000, 3: 250_000, 4: 2_000, 5: 1_000_000}[wl]
        ns = min(args.cpu_tokens or default_ns, n)
        try:
            cpu, (c_cnt, c_sums), _, _ = cpu_leg(wl, n_total, c_total, a_tok, ns, 3, 1)
        except FileNotFoundError as e:  # no fixture yet (first run): nothing to compare against
            cpu = {"value": None, "unit": UNIT, "cores": cpu_threads(), "kind": "port", "sample": f"unavailable: {e}"}
        if cpu.get("value"):
            # the same token range on the GPU, through the benched kernels (untimed): parity of the step
            run(t0 + ns)
            torch.cuda.synchronize()
            if fact:
                g_sums = out_f4.cpu().numpy()
                ok = bool(np.array_equal(g_sums, c_sums))
            else:
                g_sums = np.concatenate([v.view(4 * W, C)[:np_].cpu().numpy()
                                         for v, (W, _, _, np_) in zip(views, groups)])
                ok = bool(np.array_equal(g_sums, c_sums))
                if with_hist:
                    ok = ok and bool(np.array_equal(counts.view(L, E).cpu().numpy(), c_cnt))
            parity = {"ok": ok and fixture_match is not False, "tokens": ns, "fixture_match": fixture_match,
                      "what": (f"{'counts + ' if with_hist else ''}per-chunk hop sums of all {P_} placements over tokens "
                               f"[{a_tok}, {a_tok + ns}): the benched GPU kernels vs the CPU oracle on the same tokens "
                               f"(regenerated independently on the CPU), bit-exact")}

    # the clock poller starts before the warm-up so it is already sampling when timing begins
    sampler = ClockSampler(local).start() if rank == 0 else None
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    if with_hist and not torch.equal(counts.view(L, E), counts0):
        raise SystemExit("bench: histogram of the timed pass differs from the setup histogram")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev_a, ev_b = _events()
    ev_a.record(stream)
    for _ in range(args.steps):
        run()
    ev_b.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # the dominant kernel alone, back to back on the same stream (per-launch time for the roofline)
    ka, kb = _events()
    ka.record(stream)
    for _ in range(args.steps):
        main_kernel()
    kb.record(stream)
    torch.cuda.synchronize()
    k_ms = ka.elapsed_time(kb) / args.steps
    if sampler and world == 1:
        # a short timed region can end before the poller has a handful of samples: keep the GPU on
        # the identical (untimed) step until it has >= 8, so the reported clocks are under this load
        extra = 0
        while len(sampler.sm) < 8 and extra < 2000:
            run()
            extra += 1
            if extra % 50 == 0:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
    clocks = sampler.stop() if sampler else None
    _lib.check_err(err, "bench: device data error in the timed steps")
    if peer is not None:
        peer.check()
    t_step = torch.tensor([ev_a.elapsed_time(ev_b) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_step, op=dist.ReduceOp.MAX)
    ms = float(t_step.item())
    value = n_total * L * P_ / (ms / 1e3)

    # ---------------- roofline of the dominant kernel ----------------
    peak, peak_src = measured_peak()
    if fused:
        kname, tkey = ("mp_hist_score_u8 (fused hist+score of 4 placements; " + algo_used(True, 1) + ")"), "fused"
    elif fact:
        kname, tkey = "mp_hist_chunks_u8 (factorized evaluator: per-chunk histogram int64 [C][L][E])", "hist_chunks"
    else:
        W0 = groups[0][0]
        kname = f"mp_score_u8 (W={W0}, first of {len(groups)} launch(es) per step; {algo_used(False, W0)})"
        tkey = "score" if W0 == 1 else f"score_w{W0}"
    alg_bytes = n * L * K  # one u8 id per (token, layer, pick), per launch
    achieved = alg_bytes / (k_ms / 1e3) / 1e9
    traffic = None
    try:
        tr = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        ent = tr.get(tkey, {})
        if ent.get("tokens") and C == ent.get("chunks", C):
            traffic = ent["dram_bytes_per_launch"] * n / ent["tokens"]  # scaled to this launch's tokens
    except Exception:
        traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kname, "kernel_ms_per_launch": k_ms,
                "kernel_ms_source": f"{args.steps} back-to-back launches of the kernel alone, CUDA events on its stream",
                "kernel_share_of_step": (k_ms * (1 if fused or fact else len(groups)) / ms) if world == 1 else None,
                "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src}

    # ---------------- sustained: the same step back to back for >= --sustained-s ----------------
    sustained = None
    if world == 1 and args.sustained_s > 0:
        n_sus = max(args.steps, int(args.sustained_s * 1e3 / ms))
        smp = ClockSampler(local).start()
        sa, sb = _events()
        sa.record(stream)
        for i in range(n_sus):
            run()
            if i % 200 == 199:
                torch.cuda.synchronize()  # bound the launch queue; the events still bracket the whole run
        sb.record(stream)
        torch.cuda.synchronize()
        sclk = smp.stop()
        s_ms = sa.elapsed_time(sb) / n_sus
        sustained = {"steps": n_sus, "seconds": s_ms * n_sus / 1e3, "ms_per_step": s_ms,
                     "value": n_total * L * P_ / (s_ms / 1e3),
                     "hbm_frac": alg_bytes * (1 if fused or fact else len(groups)) / (s_ms / 1e3) / 1e9 / peak
                     if not fact else None,
                     "sm_mhz": sclk.get("sm_mhz"), "sm_min_mhz": sclk.get("sm_min_mhz"), "reasons": sclk.get("reasons")}
        roofline["frac_sustained"] = sustained["hbm_frac"]

    # ------- config 4: the 256 streaming passes beside the factorized step (bit-identical check) -------
    passes = None
    if fact:
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        run()
        torch.cuda.synchronize()
        ok = torch.equal(out_f4, buf[(L * E if with_hist else 0):][:P_ * C].view(P_, C))
        pa, pb = _events()
        n_p = max(3, args.steps // 4)
        pa.record(stream)
        for _ in range(n_p):
            step()
        pb.record(stream)
        torch.cuda.synchronize()
        p_ms = pa.elapsed_time(pb) / n_p
        passes = {"ms_per_step": p_ms, "launches_per_step": len(groups), "algorithm": "count-contract",
                  "value": n_total * L * P_ / (p_ms / 1e3), "bit_identical_to_step": ok,
                  "note": f"evaluate_many(method='count'): {len(groups)} mp_score_u8 W={groups[0][0]} passes over the resident trace"}

    # ---------------- e2e through the public API, host buffers ----------------
    e2e = None
    if not args.no_e2e:
        host_tok = trace.to_host(pin=True, layout="tokens")   # the SPEC's token-major [N, L, K] selections
        host_pl = trace.to_host(pin=True)                      # layer planes (binary sidecar form)
        cand_host = torch.from_numpy(cand).pin_memory() if fact else None
        steps_e = max(1, args.e2e_steps if wl != 5 else 1)

        def api_call(host):
            if with_hist:
                return ev.evaluate_with_stats(host, placements, costs[0])[0].counts
            if fact:  # the candidate batch as one pinned host array, as a search loop holds it
                return ev.evaluate_batch(host, cand_host, costs[0])  # auto -> factorized for P > 16
            return ev.score_sums(host, placements, costs)

        def time_api(host):
            api_call(host)  # warm-up
            evs = []
            res = None
            for _ in range(steps_e):
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize()
                a, b = _events()
                a.record(stream)
                res = api_call(host)  # H2D (streamed, overlapped) + device transpose + kernels + D2H + floats
                b.record(stream)
                torch.cuda.synchronize()
                evs.append(a.elapsed_time(b))
            if with_hist and world == 1 and not np.array_equal(res, counts0.cpu().numpy()):
                raise SystemExit("bench: e2e histogram differs")
            t_e = torch.tensor([float(np.mean(evs))], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
            return float(t_e.item())

        e_ms = time_api(host_tok)
        e_ms_planes = time_api(host_pl)
        fn = ("moeplace.eval.evaluate_with_stats(4 placements, cost)" if with_hist
              else f"moeplace.eval.evaluate_batch(int32 [{P_}, L, E] candidate batch in pinned host memory, "
                   "method='auto' -> factorized)" if fact
              else f"moeplace.eval.score_sums({P_} placements)")
        e2e = {"value": n_total * L * P_ / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(n * L * K * world + (cand.nbytes if fact else 0)),
               "d2h_bytes_per_step": int(((L * E if with_hist else 0) + P_ * C) * 8 * world),
               "api": fn + " on ActivationTrace.from_host_tokens: token-major uint8 [N, L, K] selections in pinned "
                           "host memory, streamed in 1M-token slices and transposed into layer planes on the device",
               "layer_planes_input": {"value": n_total * L * P_ / (e_ms_planes / 1e3), "ms_per_step": e_ms_planes,
                                      "api": fn + " on trace.to_host(pin=True) (layer planes, binary-sidecar form)"}}
        del host_tok, host_pl

    if rank == 0:
        cfg = workload(wl, world, n, n_total, P_)
        if args.chunks:
            cfg["workload"] += f" [--chunks {CHUNKS_PER_GPU}: {n / C:.0f} tokens per chunk]"
        engine = {"kernel_mode": "fused" if fused else "factorized" if fact else "separate",
                  "hop_sum_algorithm": (algo_used(True, 1) if fused else "factorized" if fact else
                                        "/".join(sorted({algo_used(False, W) for W, _, _, _ in groups}))),
                  "topologies": kinds, "chunks": C}
        launches = 1 if (fused or fact) else len(groups) + (1 if with_hist else 0)
        if fact:
            launches = 3  # mp_hist_chunks_u8, mp_count_digits_u8, mp_contract_tc_u8 (tcgen05 kind::i8)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
                "vs_baseline": None, "dtype": "u8", "data": "synthetic (counter-based Zipf generator, seed 0)",
                "config": cfg, "engine": engine, "roofline": roofline, "cpu_baseline": cpu, "parity": parity,
                "e2e": e2e, "gpu_launches": launches * args.steps, "clocks": clocks, "sustained": sustained,
                "passes": passes, "hbm_gbs_step": n * L * K / (ms / 1e3) / 1e9,
                # `value` counts token-layers x placements as BASELINE.json's metric names it; with
                # count-contract / factorized scoring a placement costs O(C*L*E) per (layer, chunk)
                # piece, not per token, so the per-byte rate is value / placements (and hbm_gbs_step)
                "token_layers_per_s": n_total * L / (ms / 1e3), "placements": P_,
                "value_note": "value = token-layers x placements per second (BASELINE metric); the trace "
                              "bytes processed per second are token_layers_per_s x K = hbm_gbs_step x N GPUs"}
        emit(line)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
