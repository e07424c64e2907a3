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
