"""The C-ABI library loads on a CPU-only box and exports exactly what include/moeplace_cuda.h
declares (no compute calls without a GPU, except the host solver)."""
import ctypes
import re
from pathlib import Path

import numpy as np

from paper_2508_09229_b200 import _build, _lib

ROOT = Path(__file__).resolve().parent.parent


def header_symbols():
    text = (ROOT / "include" / "moeplace_cuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mp_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_loads():
    lib = _build.build()
    assert lib.exists()
    L = _lib.load()
    assert L.mp_abi_version() == 1


def test_every_header_symbol_is_exported_and_bound():
    syms = header_symbols()
    assert len(syms) >= 15
    L = ctypes.CDLL(str(_lib.LIB_PATH))
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_status_strings_and_arg_checks():
    L = _lib.load()
    assert L.mp_status_string(0) == b"ok"
    assert b"argument" in L.mp_status_string(1)
    # argument validation is synchronous and needs no device
    assert L.mp_hist_u8(None, 0, 0, 0, 1, 1, 1, None, None, None) == 1
    assert L.mp_score_u8(None, 0, 0, 0, 1, 1, None, 1, None, 1, 0, None, None) == 1
    assert L.mp_gen_trace(0, 0, 1, 1, 1, 300, None, None, None, 16, None) == 3  # E > 256 unsupported


def test_argument_validation_matrix():
    """Every rejection is synchronous and happens before any CUDA call (fake pointers are never
    dereferenced), with the status the wrappers map to ConfigError (1/3)."""
    L = _lib.load()
    P = 0x10000  # 16-byte aligned fake device pointer
    ARG, UNS = 1, 3
    N, K, Lr, E = 100, 8, 4, 256
    st = 800  # >= N*K, multiple of 16
    cases = [
        (L.mp_hist_u8(P, st, 0, N, Lr, K, E, P, None, None), ARG),          # err required
        (L.mp_hist_u8(P + 1, st, 0, N, Lr, K, E, P, P, None), ARG),         # misaligned planes
        (L.mp_hist_u8(P, st + 8, 0, N, Lr, K, E, P, P, None), ARG),         # stride % 16
        (L.mp_hist_u8(P, 784, 0, N, Lr, K, E, P, P, None), ARG),            # stride < N*K
        (L.mp_hist_u8(P, st, 5, 4, Lr, K, E, P, P, None), ARG),             # t1 < t0
        (L.mp_hist_u8(P, st, 0, N, Lr, K, 0, P, P, None), ARG),             # E = 0
        (L.mp_hist_u8(P, st, 0, N, Lr, K, 257, P, P, None), UNS),           # E > 256
        (L.mp_hist_u8(P, st, 0, N, 0, K, E, P, P, None), ARG),              # L = 0
        (L.mp_hist_chunks_u8(P, st, 0, N, Lr, K, E, P, 0, P, P, None), ARG),  # C = 0
        (L.mp_hist_score_u8(P, st, 0, N, Lr, K, E, P, 1, P, 8, P, P, None, None), ARG),
        (L.mp_hist_score_u8(P, st, 0, N, Lr, K, E, P, 1, P, 256, P, P, P, None), UNS),
        (L.mp_score_u8(P, st, 0, N, Lr, K, P, 1, P, 3, 8, P, None), ARG),   # W not 1/2/4
        (L.mp_score_u8(P, st, 0, N, Lr, K, P, 1, P, 1, -1, P, None), ARG),
        (L.mp_score_u8(P, st, 0, N, Lr, K, P, 1, P, 1, 300, P, None), UNS),
        (L.mp_pack_tables(P, 1, P, P, 5, Lr, E, 8, P, 1, P, None), ARG),     # P > 4*W
        (L.mp_pack_tables(P, 1, P, P, 4, Lr, E, 8, P, 1, None, None), ARG),  # err required
        (L.mp_token_hops_u8(P, st, 0, N, 58, 8, P, 200, P, P, None), UNS),   # L*K*max_p > 65535
        (L.mp_apsp_bfs(P, P, 9000, P, 1, P, 1, P, P, None), UNS),
        (L.mp_apsp_bfs(P, P, 10, P, 1, P, 1, P, None, None), ARG),
        (L.mp_gen_trace(0, 0, N, 70000, K, E, P, P, P, st, None), ARG),     # grid.y limit
        (L.mp_gen_trace(0, 0, N, Lr, 9, 8, P, P, P, st, None), ARG),        # K > E
        (L.mp_score_dedup_u8(P, 33 * N + 12, 0, N, Lr, 33, P, 1, P, P, P, P, P, P, None), UNS),
        (L.mp_comm_map(P, P, P, P, 4, P, P, Lr, E, 8, P, None, None), ARG),
        (L.mp_pack_server_tables(P, 1, P, P, 5, Lr, E, 8, P, P, None), ARG),
        (L.mp_contract_counts(P, 65535 * 16 + 1, P, 1, 10, P, None), UNS),
        (L.mp_count_digits_u8(P, 4, 10, 2, 8, P, P, None), ARG),            # ldd < LE
        (L.mp_count_digits_u8(P, 4, 10, 2, 16, P, None, None), ARG),        # err required
        (L.mp_count_digits_u8(P, 4, 10, 3, 16, P, P, None), ARG),           # ndig not 1/2/4
        (L.mp_contract_tc_u8(P, 8, 24, P, 4, 2, 20, 32, P, 0, None), ARG),  # ldpe not a multiple of 16
        (L.mp_contract_tc_u8(P, 8, 32, P, 4, 3, 20, 32, P, 0, None), ARG),  # ndig not 1/2/4
        (L.mp_contract_tc_u8(P, 8, 32, P, 4, 2, 20, 32, P, -70000, None), ARG),  # absurd pair count
        (L.mp_pe_gather_u8(P, 1, Lr, 8, None, P, None, 4, E, P, Lr * E, None, None), ARG),  # err required
        (L.mp_pe_gather_u8(P, 1, Lr, 8, None, P, None, 4, E, P, Lr * E - 1, P, None), ARG),  # ldpe < L*E
        (L.mp_perturb_pe_u8(P, Lr, E, 4, 2, 0, 0, P, Lr * E + 8, P, None), ARG),  # ldpe not 16-aligned
        (L.mp_batch_objective(P, P, 4, 8, 3, 1.0, P, None), ARG),           # unknown objective kind
        (L.mp_search_accept(P, 4, P, 2, E, P, P, P, P, 0, None, None), ARG),  # accepted[] required
        (L.mp_objective_f64(P, P, 8, 16, 1, P, None), ARG),                 # ldpe < LE
        (L.mp_coeffs(P, 0, P, Lr, E, 8, 1e9, P, None, None), ARG),          # denom 0 with counts
        (L.mp_copy_planes_h2d(P, 8, P, 16, 16, 1, None), ARG),               # dst stride < width
        (L.mp_copy_planes_h2d(P, 16, P, 16, 0, 4, None), 0),                 # empty copy is a no-op
        (L.mp_hist_u8(P, st, 7, 7, Lr, K, E, P, P, None), 0),                # empty range is a no-op
    ]
    for i, (got, want) in enumerate(cases):
        assert got == want, (i, got, want)


def test_host_solver_through_abi():
    w = np.array([[[3, 1]]], dtype=np.int64)
    a = np.zeros((1, 1), np.int32)
    obj, flow = np.zeros(1, np.int64), np.zeros(1, np.int64)
    st = _lib.load().mp_solve_mcf(_lib.host_ptr(w), None, 1, 1, 2, 1, 1, _lib.host_ptr(a), _lib.host_ptr(obj),
                                  _lib.host_ptr(flow))
    assert st == 0 and a[0, 0] == 1 and obj[0] == 1 and flow[0] == 1


def test_sass_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_integration_stub_matches_the_abi():
    """The ctypes binding shown in INTEGRATION.md declares the same argument types as the library
    (so the documented drop-in binding cannot drift from include/moeplace_cuda.h)."""
    text = (ROOT / "INTEGRATION.md").read_text()
    names = {"_p": ctypes.c_void_p, "_i32": ctypes.c_int, "_i64": ctypes.c_int64, "C.c_char_p": ctypes.c_char_p}
    found = re.findall(r"_lib\.(mp_\w+)\.argtypes = \[(.*?)\]", text)
    assert len(found) >= 3
    for name, args in found:
        got = [names[a.strip()] for a in args.split(",")]
        assert got == list(_lib.SIGNATURES[name][1]), name


def test_auto_algorithm_rule():
    """mp_choose_algo (host-only) is the rule MP_ALGO_AUTO applies: the crossovers measured for R1
    (profiles/r2_crossovers.txt) -- count-contract / gather for long chunks, the segmented
    gather for dialog-length ones, the token walk only for the shortest score-only chunks."""
    N, L, K = 10_000_000, 58, 8
    tpc = {150: 66_667, 1500: 6667, 2000: 5000, 2500: 4000, 71_429: 140, 150_000: 67, 250_000: 40}
    want = {  # (hist, W): algorithm per chunk count
        (True, 1): {150: "count", 1500: "count", 2000: "count", 2500: "seg", 71_429: "seg", 150_000: "seg"},
        (False, 1): {150: "gather", 1500: "seg", 2000: "seg", 71_429: "seg", 150_000: "seg", 250_000: "token"},
        (False, 4): {150: "count", 1500: "count", 2000: "count", 71_429: "seg", 150_000: "seg"},
        (True, 4): {150: "count", 1500: "count", 2000: "count", 71_429: "seg", 150_000: "seg"},
    }
    for (hist, W), row in want.items():
        for C, algo in row.items():
            assert _lib.choose_algo(hist, W, N, C, L, K, 8) == algo, (hist, W, C, tpc[C])
    # SEG needs K = 8 and costs <= 31; otherwise the token walk / streaming algorithms apply
    assert _lib.choose_algo(False, 1, N, 71_429, L, K, 40) in ("token", "gather")
    assert _lib.choose_algo(True, 1, N, 150, L, 6, 8) == "count"
    # 32 placements per pass (W = 8): the count-contract kernel at every shape
    assert _lib.choose_algo(False, 8, N, 71_429, L, K, 8) == "count"
    assert _lib.choose_algo(True, 8, N, 150, L, K, 8) == "count"


def test_pass_lanes_rule():
    """eval.pass_lanes (host-only): 32 placements per pass where the library's AUTO picks the
    count-contract kernel (long chunks) or count is forced, 16 otherwise."""
    import types

    import torch

    from paper_2508_09229_b200 import eval as ev
    from paper_2508_09229_b200.model_trace import ModelSpec
    from paper_2508_09229_b200.placement import CostMatrix
    m = ModelSpec(58, 256, 8)
    cost = CostMatrix(torch.full((58, 32), 6, dtype=torch.uint8))
    long_chunks = types.SimpleNamespace(model=m, n_tokens=10_000_000, n_chunks=150)
    dialog = types.SimpleNamespace(model=m, n_tokens=10_000_000, n_chunks=71_429)
    assert ev.pass_lanes(long_chunks, cost) == 32
    assert ev.pass_lanes(long_chunks, [cost] * 3, hist=True) == 32
    assert ev.pass_lanes(dialog, cost) == 16
    assert ev.pass_lanes(dialog, cost, "count") == 32
    assert ev.pass_lanes(long_chunks, cost, "gather") == 16
    assert ev._lanes_for(4) == 1 and ev._lanes_for(16) == 4 and ev._lanes_for(17) == 8 and ev._lanes_for(32) == 8
