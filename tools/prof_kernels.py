"""Profiling driver: builds the bench's config-2 trace (R1, 10M tokens) and launches each
streaming kernel variant a few times, so ncu can capture them by name.
  python tools/prof_kernels.py [--tokens N] [--reps R]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import moeplace.eval as ev  # noqa: E402
import moeplace.model_trace as mt  # noqa: E402
import moeplace.placement as mpl  # noqa: E402
import moeplace.topology as topo  # noqa: E402
from paper_2508_09229_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=10_000_000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--which", default="fused,hist,score1,score4,fused_gather,score4_gather")
ap.add_argument("--chunks", type=int, default=150)
a = ap.parse_args()
L, E, K = 58, 256, 8
m = mt.ModelSpec(L, E, K)
g = topo.build_topology(topo.TopologySpec("FatTree", 8, 4, 8, {"spines": 4}))
d = topo.all_pairs_hops(g)
order = topo.locality_order(g, d)
attn = mt.default_attention_placement(m, order)
cost = mpl.cost_matrix(d, attn)
c = mpl.Constraints(64, 1)
pls = [mpl.place_round_robin(m, attn, order, c), mpl.place_greedy(m, attn, cost, c)] * 8
tr = mt.generate_trace(m, 1.2, a.tokens, a.chunks, 0)
P, st = tr.planes, tr.planes.shape[1]
C = tr.n_chunks
b = _lib.to_dev(tr.chunk_bounds, torch.int64)
t1, mp1 = ev._group_tables(pls[:4], [cost] * 4, m, 1)
t4, mp4 = ev._group_tables(pls[:16], [cost] * 16, m, 4)
cnt = torch.zeros(L * E, dtype=torch.int64, device="cuda")
s = torch.zeros(16 * C, dtype=torch.int64, device="cuda")
err = _lib.new_err()
sh = _lib.stream_handle()
srv1 = torch.empty((L, 256), dtype=torch.int32, device="cuda")
_lib.call("mp_pack_server_tables", _lib.ptr(_lib.to_dev(g.device_server[None].astype("int32"), torch.int32)), 1,
          _lib.ptr(_lib.to_dev(__import__("numpy").stack([p.assign for p in pls[:4]]), torch.int32)),
          _lib.ptr(torch.zeros(4, dtype=torch.int32, device="cuda")), 4, L, E, g.n_devices, _lib.ptr(srv1),
          _lib.ptr(err), sh)
src1 = _lib.to_dev(__import__("numpy").tile(g.device_server[attn.dispatch].astype("uint8"), (4, 1)), torch.uint8)
s2 = torch.zeros(4 * C, dtype=torch.int64, device="cuda")
s3 = torch.zeros(4 * C, dtype=torch.int64, device="cuda")
for _ in range(a.reps):
    for w in a.which.split(","):
        if w == "fused":
            _lib.call("mp_hist_score_u8", _lib.ptr(P), st, 0, a.tokens, L, K, E, _lib.ptr(b), C, _lib.ptr(t1), mp1,
                      _lib.ptr(cnt), _lib.ptr(s), _lib.ptr(err), sh)
        elif w == "hist":
            _lib.call("mp_hist_u8", _lib.ptr(P), st, 0, a.tokens, L, K, E, _lib.ptr(cnt), _lib.ptr(err), sh)
        elif w == "score1":
            _lib.call("mp_score_u8", _lib.ptr(P), st, 0, a.tokens, L, K, _lib.ptr(b), C, _lib.ptr(t1), 1, mp1,
                      _lib.ptr(s), sh)
        elif w == "fused_gather":
            _lib.call("mp_hist_score_ex_u8", _lib.ptr(P), st, 0, a.tokens, L, K, E, _lib.ptr(b), C, _lib.ptr(t1), 1,
                      mp1, _lib.ptr(cnt), _lib.ptr(s), _lib.ptr(err), 1, sh)
        elif w == "score4_gather":
            _lib.call("mp_score_ex_u8", _lib.ptr(P), st, 0, a.tokens, L, K, _lib.ptr(b), C, _lib.ptr(t4), 4, mp4,
                      _lib.ptr(s), 1, sh)
        elif w in ("score1_seg", "score4_seg", "fused_seg", "fused4_seg"):  # forced MP_ALGO_SEG (4)
            W = 4 if "4" in w else 1
            t_, mp_ = (t4, mp4) if W == 4 else (t1, mp1)
            if w.startswith("fused"):
                _lib.call("mp_hist_score_ex_u8", _lib.ptr(P), st, 0, a.tokens, L, K, E, _lib.ptr(b), C, _lib.ptr(t_), W,
                          mp_, _lib.ptr(cnt), _lib.ptr(s), _lib.ptr(err), 4, sh)
            else:
                _lib.call("mp_score_ex_u8", _lib.ptr(P), st, 0, a.tokens, L, K, _lib.ptr(b), C, _lib.ptr(t_), W, mp_,
                          _lib.ptr(s), 4, sh)
        elif w == "hist_chunks":
            cc = torch.zeros((C, L * E), dtype=torch.int64, device="cuda")
            _lib.call("mp_hist_chunks_u8", _lib.ptr(P), st, 0, a.tokens, L, K, E, _lib.ptr(b), C, _lib.ptr(cc),
                      _lib.ptr(err), sh)
        elif w == "dedup":
            _lib.call("mp_score_dedup_u8", _lib.ptr(P), st, 0, a.tokens, L, K, _lib.ptr(b), C, _lib.ptr(t1),
                      _lib.ptr(srv1), _lib.ptr(src1), _lib.ptr(s), _lib.ptr(s2), _lib.ptr(s3), sh)
        elif w == "score4":
            _lib.call("mp_score_u8", _lib.ptr(P), st, 0, a.tokens, L, K, _lib.ptr(b), C, _lib.ptr(t4), 4, mp4,
                      _lib.ptr(s), sh)
torch.cuda.synchronize()
print("prof_kernels done")
