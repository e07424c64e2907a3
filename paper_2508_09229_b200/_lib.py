"""ctypes binding of libmoeplace_cuda.so (the C-ABI in include/moeplace_cuda.h) and the small
device plumbing the hot-path wrappers share.

There is no CPU fallback: if the library is missing, or no CUDA device is visible, the hot-path
operations raise ``RuntimeError`` instead of silently computing on the host.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import ConfigError, MoeplaceError

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libmoeplace_cuda.so"
if os.environ.get("MOEPLACE_EXPERIMENT_LIB"):  # tools/ only: an experimental build of the same sources
    LIB_PATH = Path(os.environ["MOEPLACE_EXPERIMENT_LIB"])

_p = C.c_void_p
_i32, _i64, _u64, _dbl = C.c_int, C.c_int64, C.c_uint64, C.c_double

# symbol -> (restype, argtypes); must list every function declared in include/moeplace_cuda.h
SIGNATURES = {
    "mp_abi_version": (_i32, []),
    "mp_status_string": (C.c_char_p, [_i32]),
    "mp_gen_trace": (_i32, [_u64, _i64, _i64, _i32, _i32, _i32, _p, _p, _p, _i64, _p]),
    "mp_validate_u8": (_i32, [_p, _i64, _i64, _i64, _i32, _i32, _i32, _p, _p]),
    "mp_count_newlines": (_i32, [_p, _i64, _p, _p]),
    "mp_find_newlines": (_i32, [_p, _i64, _p, _p, _p]),
    "mp_parse_trace_text": (_i32, [_p, _p, _i64, _i64, _i32, _i32, _i32, _p, _i64, _p, _p, _p]),
    "mp_format_lengths": (_i32, [_p, _i64, _i64, _i64, _i32, _i32, _p, _p, _p]),
    "mp_format_trace_text": (_i32, [_p, _i64, _i64, _i64, _i32, _i32, _p, _p, _p, _p]),
    "mp_hist_u8": (_i32, [_p, _i64, _i64, _i64, _i32, _i32, _i32, _p, _p, _p]),
    "mp_hist_chunks_u8": (_i32, [_p, _i64, _i64, _i64, _i32, _i32, _i32, _p, _i32, _p, _p, _p]),
    "mp_contract_counts": (_i32, [_p, _i32, _p, _i32, _i64, _p, _p]),
    "mp_count_digits_u8": (_i32, [_p, _i32, _i64, _i32, _i64, _p, _p, _p]),
    "mp_contract_tc_u8": (_i32, [_p, _i32, _i64, _p, _i32, _i32, _i64, _i64, _p, _i32, _p]),
    "mp_pack_tables": (_i32, [_p, _i32, _p, _p, _i32, _i32, _i32, _i32, _p, _i32, _p, _p]),
    "mp_score_u8": (_i32, [_p, _i64, _i64, _i64, _i32, _i32, _p, _i32, _p, _i32, _i32, _p, _p]),
    "mp_token_hops_u8": (_i32, [_p, _i64, _i64, _i64, _i32, _i32, _p, _i32, _p, _p, _p]),
    "mp_hist_score_u8": (_i32, [_p, _i64, _i64, _i64, _i32, _i32, _i32, _p, _i32, _p, _i32, _p, _p, _p, _p]),
    "mp_score_ex_u8": (_i32, [_p, _i64, _i64, _i64, _i32, _i32, _p, _i32, _p, _i32, _i32, _p, _i32, _p]),
    "mp_hist_score_ex_u8": (_i32, [_p, _i64, _i64, _i64, _i32, _i32, _i32, _p, _i32, _p, _i32, _i32, _p, _p, _p, _i32,
                                   _p]),
    "mp_choose_algo": (_i32, [_i32, _i32, _i64, _i32, _i32, _i32, _i32]),
    "mp_allreduce_peers_i64": (_i32, [_p, _i64, _p, _p, _p, _i32, _i32, C.c_uint32, _p, _p]),
    "mp_score_dedup_u8": (_i32, [_p, _i64, _i64, _i64, _i32, _i32, _p, _i32, _p, _p, _p, _p, _p, _p, _p]),
    "mp_pack_server_tables": (_i32, [_p, _i32, _p, _p, _i32, _i32, _i32, _i32, _p, _p, _p]),
    "mp_apsp_bfs": (_i32, [_p, _p, _i32, _p, _i32, _p, _i32, _p, _p, _p]),
    "mp_expand_dist": (_i32, [_p, _i32, _p, _i32, _p, _p]),
    "mp_cost_matrix": (_i32, [_p, _i32, _p, _i32, _p, _p, _i32, _p, _p]),
    "mp_coeffs": (_i32, [_p, _i64, _p, _i32, _i32, _i32, _dbl, _p, _p, _p]),
    "mp_comm_map": (_i32, [_p, _p, _p, _p, _i32, _p, _p, _i32, _i32, _i32, _p, _p, _p]),
    "mp_copy_planes_h2d": (_i32, [_p, _i64, _p, _i64, _i64, _i32, _p]),
    "mp_pe_gather_u8": (_i32, [_p, _i32, _i32, _i32, _p, _p, _p, _i32, _i32, _p, _i64, _p, _p]),
    "mp_perturb_pe_u8": (_i32, [_p, _i32, _i32, _i32, _i32, _u64, _i64, _p, _i64, _p, _p]),
    "mp_batch_objective": (_i32, [_p, _p, _i32, _i32, _i32, _dbl, _p, _p]),
    "mp_search_accept": (_i32, [_p, _i32, _p, _i32, _i32, _p, _p, _p, _p, _i64, _p, _p]),
    "mp_objective_f64": (_i32, [_p, _p, _i64, _i64, _i32, _p, _p]),
    "mp_tokens_to_planes_u8": (_i32, [_p, _i64, _i32, _i32, _p, _i64, _i64, _p]),
    "mp_solve_mcf": (_i32, [_p, _p, _i32, _i32, _i32, _i32, _i32, _p, _p, _p]),
}

MP_OK, MP_ERR_ARG, MP_ERR_CUDA, MP_ERR_UNSUPPORTED, MP_INFEASIBLE = 0, 1, 2, 3, 4
DATA_EXPERT_RANGE, DATA_DUPLICATE, DATA_UNREACHABLE, DATA_UNPLACED, DATA_HOPS_RANGE = 1, 2, 3, 4, 5

_lib = None


def load() -> C.CDLL:
    """Load the engine library (does not touch the GPU)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is not built; run `python -m paper_2508_09229_b200._build` "
                "(the moeplace hot path has no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def call(name: str, *args) -> int:
    """Invoke a C-ABI function; map synchronous failures onto the package's exceptions."""
    st = getattr(load(), name)(*args)
    if st in (MP_OK, MP_INFEASIBLE) and name == "mp_solve_mcf":
        return st
    if st == MP_OK:
        return st
    msg = f"{name}: {load().mp_status_string(st).decode()}"
    if st in (MP_ERR_ARG, MP_ERR_UNSUPPORTED):
        raise ConfigError(msg)
    raise RuntimeError(msg)


def choose_algo(hist: bool, W: int, tokens: int, C: int, L: int, K: int, max_p: int) -> str:
    """The hop-sum algorithm MP_ALGO_AUTO resolves to for this shape (mp_choose_algo; host-only)."""
    code = load().mp_choose_algo(int(hist), W, tokens, C, L, K, max_p)
    return {1: "gather", 2: "count", 3: "token", 4: "seg"}[code]


# ---- torch device plumbing -----------------------------------------------------------------

def torch():
    import torch as _t
    return _t


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("the moeplace hot path runs on a CUDA device (B200, sm_100a); none is visible "
                           "and there is no CPU fallback")
    load()
    return t.device("cuda", t.cuda.current_device())


def stream_handle():
    t = torch()
    return C.c_void_p(t.cuda.current_stream().cuda_stream)


def ptr(x):
    """Device pointer of a contiguous CUDA tensor (None -> NULL)."""
    if x is None:
        return None
    if not x.is_cuda:
        raise ConfigError("expected a CUDA tensor")
    if not x.is_contiguous():
        raise ConfigError("expected a contiguous tensor")
    return C.c_void_p(x.data_ptr())


def ptr_any(x):
    """Device pointer of a CUDA tensor whose layout the callee describes itself (pitch argument)."""
    if not x.is_cuda:
        raise ConfigError("expected a CUDA tensor")
    return C.c_void_p(x.data_ptr())


def to_dev(a, dtype):
    """numpy array / torch tensor -> contiguous CUDA tensor of `dtype`."""
    t = torch()
    dev = require_cuda()
    if isinstance(a, t.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return t.as_tensor(np.ascontiguousarray(a), device=dev).to(dtype).contiguous()


def new_err():
    t = torch()
    return t.zeros(4, dtype=t.int64, device=require_cuda())


def read_err(err) -> tuple[int, int, int, int]:
    v = err.cpu().tolist()
    return int(v[0]), int(v[1]), int(v[2]), int(v[3])


def check_err(err, what: str, exc=MoeplaceError):
    code, a, b, n = read_err(err)
    if code == 0:
        return
    if code == DATA_EXPERT_RANGE:
        raise exc(f"{what}: expert id {b} out of range in layer {a} ({n} occurrences)")
    if code == DATA_UNPLACED:
        raise exc(f"{what}: expert ({a}, {b}) is not placed on a valid device ({n} entries)")
    raise exc(f"{what}: device data error code {code} ({a}, {b}, x{n})")


def host_ptr(a: np.ndarray):
    if not a.flags.c_contiguous:
        raise ConfigError("expected a C-contiguous array")
    return a.ctypes.data_as(C.c_void_p)
