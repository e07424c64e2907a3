"""Times each streaming kernel variant on the config-2 trace (R1, 10M tokens) with CUDA events.
  python tools/time_kernels.py [--tokens N] [--reps R] [--s zipf]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import moeplace.eval as ev  # noqa: E402
import moeplace.model_trace as mt  # noqa: E402
import moeplace.placement as mpl  # noqa: E402
import moeplace.topology as topo  # noqa: E402
from paper_2508_09229_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=10_000_000)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--s", type=float, default=1.2)
ap.add_argument("--out")
ap.add_argument("--lib", help="load this libmoeplace_cuda.so variant instead of the product build")
ap.add_argument("--only", default="")
ap.add_argument("--chunks", type=int, default=150)
ap.add_argument("--dump", help="save each kernel's hop sums / counts (zeroed before it runs) to this .npz")
a = ap.parse_args()
if a.lib:
    from pathlib import Path
    _lib.LIB_PATH = Path(a.lib)
L, E, K = 58, 256, 8
m = mt.ModelSpec(L, E, K)
g = topo.build_topology(topo.TopologySpec("FatTree", 8, 4, 8, {"spines": 4}))
d = topo.all_pairs_hops(g)
order = topo.locality_order(g, d)
attn = mt.default_attention_placement(m, order)
cost = mpl.cost_matrix(d, attn)
c = mpl.Constraints(64, 1)
pls = [mpl.place_round_robin(m, attn, order, c), mpl.place_greedy(m, attn, cost, c)] * 16
tr = mt.generate_trace(m, a.s, a.tokens, a.chunks, 0)
P, st = tr.planes, tr.planes.shape[1]
C = tr.n_chunks
b = _lib.to_dev(tr.chunk_bounds, torch.int64)
tabs = {W: ev._group_tables(pls[:4 * W], [cost] * 4 * W, m, W) for W in (1, 2, 4, 8)}
cnt = torch.zeros(L * E, dtype=torch.int64, device="cuda")
s = torch.zeros(32 * C, dtype=torch.int64, device="cuda")
err = _lib.new_err()
sh = _lib.stream_handle()


def run(w):
    """fused / hist / scoreW (library's algorithm) and fused_gather / scoreW_gather (forced gather)."""
    algo = 0
    for suf, code in (("_gather", 1), ("_count", 2), ("_token", 3), ("_seg", 4)):
        if w.endswith(suf):
            algo, w = code, w[:-len(suf)]
    if w.startswith("fused"):  # fused = histogram + 4 placements; fused2 / fused4 = + 8 / 16 placements
        Wf = int(w[5:] or 1)
        t, mp_ = tabs[Wf]
        _lib.call("mp_hist_score_ex_u8", _lib.ptr(P), st, 0, a.tokens, L, K, E, _lib.ptr(b), C, _lib.ptr(t), Wf, mp_,
                  _lib.ptr(cnt), _lib.ptr(s), _lib.ptr(err), algo, sh)
    elif w == "hist":
        _lib.call("mp_hist_u8", _lib.ptr(P), st, 0, a.tokens, L, K, E, _lib.ptr(cnt), _lib.ptr(err), sh)
    else:
        W = int(w[-1])
        t, mp_ = tabs[W]
        _lib.call("mp_score_ex_u8", _lib.ptr(P), st, 0, a.tokens, L, K, _lib.ptr(b), C, _lib.ptr(t), W, mp_,
                  _lib.ptr(s), algo, sh)


hops_out = torch.empty((4, a.tokens), dtype=torch.int32, device="cuda")
rep_scratch = torch.empty((L, 256, 32), dtype=torch.int32, device="cuda")
cc = torch.zeros((C, L * E), dtype=torch.int64, device="cuda")
srv_t = torch.empty((L, 256), dtype=torch.int32, device="cuda")
_lib.call("mp_pack_server_tables", _lib.ptr(_lib.to_dev(g.device_server[None].astype("int32"), torch.int32)), 1,
          _lib.ptr(_lib.to_dev(__import__("numpy").stack([p.assign for p in pls[:4]]), torch.int32)),
          _lib.ptr(torch.zeros(4, dtype=torch.int32, device="cuda")), 4, L, E, g.n_devices, _lib.ptr(srv_t),
          _lib.ptr(err), sh)
src = _lib.to_dev(__import__("numpy").tile(g.device_server[attn.dispatch].astype("uint8"), (4, 1)), torch.uint8)
dd = torch.zeros((3, 4, C), dtype=torch.int64, device="cuda")


def run_ext(w):
    t1_, mp1_ = tabs[1]
    if w == "token_hops":
        _lib.call("mp_token_hops_u8", _lib.ptr(P), st, 0, a.tokens, L, K, _lib.ptr(t1_), mp1_, _lib.ptr(rep_scratch),
                  _lib.ptr(hops_out), sh)
    elif w == "hist_chunks":
        _lib.call("mp_hist_chunks_u8", _lib.ptr(P), st, 0, a.tokens, L, K, E, _lib.ptr(b), C, _lib.ptr(cc),
                  _lib.ptr(err), sh)
    elif w == "dedup":
        _lib.call("mp_score_dedup_u8", _lib.ptr(P), st, 0, a.tokens, L, K, _lib.ptr(b), C, _lib.ptr(t1_),
                  _lib.ptr(srv_t), _lib.ptr(src), _lib.ptr(dd[0]), _lib.ptr(dd[1]), _lib.ptr(dd[2]), sh)


# roofline denominator: the driver-measured HBM copy bandwidth (MEASURED_PEAKS.json), else the recipe's
_pk = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
PEAK = float(json.load(open(_pk)).get("hbm_gbs", 6458.4)) if os.path.exists(_pk) else 6458.4
res = {}
dumps = {}
bytes_ = a.tokens * L * K
for w in (a.only.split(",") if a.only else ("hist", "score1", "score2", "score4", "fused", "token_hops", "hist_chunks", "dedup")):
    base = w
    for suf in ("_gather", "_count", "_token", "_seg"):
        base = base[:-len(suf)] if base.endswith(suf) else base
    fn = run if base in ("hist", "score1", "score2", "score4", "score8", "fused", "fused2", "fused4", "fused8") else run_ext
    s.zero_()
    cnt.zero_()
    fn(w)
    torch.cuda.synchronize()
    if a.dump:
        dumps[w + "_sums"] = s.cpu().numpy().copy()
        dumps[w + "_counts"] = cnt.cpu().numpy().copy()
    for _ in range(2):
        fn(w)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(w)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.mean(ts))
    res[w] = {"ms": ms, "min_ms": float(min(ts)), "GBps": bytes_ / ms / 1e6, "frac_hbm": bytes_ / ms / 1e6 / PEAK}
    print(f"{w:8s} {ms:7.3f} ms (min {min(ts):.3f})  {bytes_ / ms / 1e6:8.1f} GB/s  {100 * bytes_ / ms / 1e6 / PEAK:5.1f}%")
if a.dump:
    np.savez(a.dump, **dumps)
if a.only:
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)
    sys.exit(0)
# device text IO at 1M tokens (text ~2.1 KB per R1 token)
import tempfile, time  # noqa: E401,E402
sub = tr.view(0, 15)  # first 15 chunks (~1M tokens)
with tempfile.TemporaryDirectory() as d:
    f = os.path.join(d, "t.txt")
    mt.write_trace(sub, f, engine="cuda")
    torch.cuda.synchronize()
    t_a = time.perf_counter()
    mt.write_trace(sub, f, engine="cuda")
    t_w = time.perf_counter() - t_a
    size = os.path.getsize(f)
    mt.parse_trace(f)
    torch.cuda.synchronize()
    t_a = time.perf_counter()
    back = mt.parse_trace(f)
    torch.cuda.synchronize()
    t_p = time.perf_counter() - t_a
    ok = bool((back.tokens()[:1000] == sub.tokens()[:1000]).all())
res["io"] = {"tokens": sub.n_tokens, "text_bytes": size, "write_s": t_w, "parse_s": t_p, "roundtrip_ok": ok,
             "write_GBps": size / t_w / 1e9, "parse_GBps": size / t_p / 1e9}
print("io", res["io"])
if a.out:
    json.dump(res, open(a.out, "w"), indent=1)
