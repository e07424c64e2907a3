"""Wall time of the reference-facing pipeline (moeplace.cli.run_experiment) on BASELINE configs 1
and 3 (R1, 10M tokens, the four SPEC topologies), with a per-stage breakdown from cProfile's
top entries.  Not product code: a measurement driver for DESIGN.md.
  python tools/time_pipeline.py [--r1-tokens N]"""
import argparse
import cProfile
import os
import pstats
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import moeplace.cli as cli  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--r1-tokens", type=int, default=10_000_000)
ap.add_argument("--profile", action="store_true")
a = ap.parse_args()

CFG1 = {"model": "16b", "L": 27, "E": 64, "K": 6, "c_exp": 54, "c_layer": 2, "topology": "FatTree",
        "num_leaf_switches": 2, "num_nodes_per_leaf": 2, "num_gpus_per_server": 8, "spines": 4,
        "zipf_s": 1.2, "n_tokens": 1_000_000, "n_chunks": 150, "seed": 0, "train_chunks": 100, "test_chunks": 50}
CFG3 = {"model": "r1", "L": 58, "E": 256, "K": 8, "c_exp": 64, "c_layer": 1,
        "topologies": ["FatTree", "FatTreeHier", "Dragonfly", "DragonflySparse"],
        "num_leaf_switches": 16, "num_nodes_per_leaf": 4, "num_gpus_per_server": 4,
        "zipf_s": 1.2, "n_tokens": a.r1_tokens, "n_chunks": 150, "seed": 0, "train_chunks": 100, "test_chunks": 50}

for name, cfg in (("config1 (16B, 1M tokens, FatTree 2x2x8)", CFG1),
                  (f"config3 (R1, {a.r1_tokens} tokens, 4 topologies 16x4x4)", CFG3)):
    with tempfile.TemporaryDirectory() as d:
        cfg = dict(cfg, output_dir=d)
        cli.run_experiment(dict(cfg, output_dir=os.path.join(d, "warm"), n_tokens=20000))  # warm-up
        prof = cProfile.Profile() if a.profile else None
        t0 = time.perf_counter()
        if prof:
            prof.enable()
        res = cli.run_experiment(cfg)
        if prof:
            prof.disable()
        dt = time.perf_counter() - t0
        print(f"{name}: run_experiment {dt:.2f} s")
        for row in res["rows"]:
            print("   ", row)
        if prof:
            pstats.Stats(prof).sort_stats("cumulative").print_stats(18)
