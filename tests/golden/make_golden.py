"""Generate the golden fixtures under tests/golden/ (run here, in the build container, where
/root/reference exists; the fixtures are committed and nothing reads /root/reference at test
time).

  gain_kat.json        the 48 (RR, method, printed gain) cells of PAPER.md Tables 2, 3a, 3b, 4
                       (PAPER.md:363-381, 402-420, 434-452, 577-595): KATs for gain()
  spec_examples.json   the SPEC.md known-answer examples for the hot-path operations, restated
                       as concrete inputs/outputs (each entry cites its SPEC line)
  oracle_small.npz     a frozen oracle run (generator + counts + RR/greedy chunk sums on a small
                       FatTree): regression fixture tying the oracle, the GPU and this file

Usage: python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import re
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
PAPER = Path("/root/reference/PAPER.md")

ROW = re.compile(r"^\s*(FatTree|Dragonfly|Sparse)?\s*&\s*(RR|Greedy|ILP|ILPLoad)\s*&\s*(?:\\textbf\{)?([0-9.]+)\}?±([0-9.]+)"
                 r"\s*&\s*(?:\\textbf\{)?(-?[0-9.]*)\\?%?")


def gain_cells():
    lines = PAPER.read_text().splitlines()
    tables = {"table2": (363, 381), "table3a": (402, 420), "table3b": (434, 452), "table4": (577, 595)}
    out = []
    for name, (a, b) in tables.items():
        rr = None
        block = 0
        for ln in range(a, b + 1):
            m = ROW.match(lines[ln - 1])
            if not m:
                continue
            method, hops, pct = m.group(2), float(m.group(3)), m.group(5)
            if method == "RR":
                rr = hops
                block += 1
                continue
            out.append({"table": name, "block": block, "line": ln, "method": method, "rr_hops": rr,
                        "method_hops": hops, "gain_pct": float(pct)})
    return out


def spec_examples():
    """Concrete restatements of SPEC.md examples (inputs small enough to verify by hand)."""
    return {
        # 1 token, L=1, K=2, experts {0,1}, E=4 -> f = [0.5, 0.5, 0, 0]
        "freq_one_token": {"L": 1, "E": 4, "K": 2, "tokens": [[[0, 1]]], "f": [[0.5, 0.5, 0.0, 0.0]],
                           "cite": "SPEC.md:146"},
        # every token selects the same K set -> those at 1/K, rest 0
        "freq_same_set": {"L": 2, "E": 6, "K": 3, "tokens": [[[5, 1, 2], [0, 3, 4]]] * 7,
                          "f": [[0, 1 / 3, 1 / 3, 0, 0, 1 / 3], [1 / 3, 0, 0, 1 / 3, 1 / 3, 0]],
                          "cite": "SPEC.md:147"},
        # L=1, K=2, placed p-values {4, 2} -> 6
        "token_hops_4_2": {"p": [[4, 2]], "assign": [[0, 1]], "selection": [[0, 1]], "hops": 6,
                           "cite": "SPEC.md:343"},
        # everything colocated with d=c -> 0
        "token_hops_colocated": {"p": [[0, 4, 4]], "assign": [[0, 0, 0]], "selection": [[0, 2]], "hops": 0,
                                 "cite": "SPEC.md:342"},
        # FatTree 2 leaves x 1 server x 1 GPU, 1 spine -> dist 4
        "fattree_2leaf": {"kind": "FatTree", "leaves": 2, "spl": 1, "gps": 1, "extra": {"spines": 1},
                          "dist": [[0, 4], [4, 0]], "cite": "SPEC.md:48,59"},
        # 1 leaf, 1 server, 4 GPUs -> all zero
        "one_server": {"kind": "Dragonfly", "leaves": 1, "spl": 1, "gps": 4, "extra": {},
                       "dist": [[0] * 4] * 4, "cite": "SPEC.md:49,57"},
        # two servers under the same leaf -> 2
        "same_leaf": {"kind": "FatTree", "leaves": 1, "spl": 2, "gps": 1, "extra": {"spines": 1},
                      "dist": [[0, 2], [2, 0]], "cite": "SPEC.md:58"},
        # 2-leaf FatTree, d on A, c on B, s = A's server -> p = 0 + 4
        "cost_cross_leaf": {"kind": "FatTree", "leaves": 2, "spl": 1, "gps": 1, "extra": {"spines": 1},
                            "dispatch": [0], "collect": [1], "p": [[4, 4]], "cite": "SPEC.md:206"},
        # solver KATs
        "solve_1x1x2": {"w": [[[3, 1]]], "c_layer": 1, "c_exp": 1, "assign": [[1]], "objective": 1,
                        "cite": "SPEC.md:288"},
        "solve_1x2x2": {"w": [[[0, 5], [0, 5]]], "c_layer": 1, "c_exp": 1, "objective": 5, "cite": "SPEC.md:289"},
        # greedy L=1,E=2,S=2,c_layer=1,p=[0,4] -> e0 on 0, e1 on 1, cost 4
        "greedy_2x2": {"p": [[0, 4]], "c_layer": 1, "c_exp": 2, "assign": [[0, 1]], "cost": 4, "cite": "SPEC.md:232"},
        # gain KATs
        "gain": [[5003.98, 4391.73, 13.9], [5003.98, 4755.52, 5.2], [3757.23, 3280.58, 14.5]],
        # L=4, 4 devices -> dispatch = order[0..3], collect = order[1..3, 3]
        "attention_L4": {"L": 4, "order": [3, 1, 2, 0], "dispatch": [3, 1, 2, 0], "collect": [1, 2, 0, 0],
                         "cite": "SPEC.md:120"},
        # RR circular window, dispatch at position 0 with d = 4 -> {n-2, n-1, 0, 1}
        "rr_wrap": {"E": 4, "c_layer": 1, "n": 8, "positions": [6, 7, 0, 1], "cite": "SPEC.md:224"},
        # SPEC.md:155-157 split examples
        "split": {"cases": [[150, 100, 50, True], [2, 1, 1, True], [4, 3, 3, False]], "cite": "SPEC.md:155-157"},
    }


def oracle_small():
    sys.path.insert(0, str(ROOT))
    from oracle import gen, stats, evaluate, topology
    L, E, K, N, C, seed = 27, 64, 6, 3000, 15, 7
    sel, bounds = gen.generate(L, E, K, 1.2, N, C, seed)
    cnt = stats.counts(sel, E)
    # small FatTree: 2 leaves x 2 servers x 8 GPUs, 4 spines; servers 0,1 on leaf node 4, 2,3 on leaf 5
    links = [(0, 4), (1, 4), (2, 5), (3, 5)] + [(lf, sp) for lf in (4, 5) for sp in (6, 7, 8, 9)]
    dsrv = topology.server_hops(10, links, 4)
    dev_srv = np.repeat(np.arange(4), 8)
    disp = np.array([(l * 32) // L for l in range(L)])
    coll = np.concatenate([disp[1:], disp[-1:]])
    p = topology.cost_matrix(dsrv, dev_srv, disp, coll)
    rng = np.random.default_rng(seed)
    assign = np.stack([rng.permutation(np.repeat(np.arange(32), 2)) for _ in range(L)]).astype(np.int32)
    pe = evaluate.pe_table(p, assign)
    sums = evaluate.chunk_sums(sel, pe, bounds)
    np.savez_compressed(HERE / "oracle_small.npz", L=L, E=E, K=K, N=N, C=C, seed=seed, zipf_s=1.2,
                        sel=sel, bounds=bounds, counts=cnt, dsrv=dsrv, p=p, assign=assign, sums=sums)


if __name__ == "__main__":
    cells = gain_cells()
    assert len(cells) == 48, len(cells)
    (HERE / "gain_kat.json").write_text(json.dumps(cells, indent=1))
    (HERE / "spec_examples.json").write_text(json.dumps(spec_examples(), indent=1))
    oracle_small()
    print("wrote", len(cells), "gain cells, spec examples, oracle_small.npz")
