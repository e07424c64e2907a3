"""In-tree build of libmoeplace_cuda.so (sm_100a) with nvcc.

The shared library travels with the repo snapshot to the GPU box (it is git-ignored, not
gpurun-ignored), so the product never depends on a JIT cache.  ``python -m
paper_2508_09229_b200._build`` or ``__graft_entry__.build()`` runs this.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libmoeplace_cuda.so"
ROOT = PKG.parent

CU_SOURCES = ["stream.cu", "seg.cu", "gen.cu", "topo.cu", "dedup.cu", "parse.cu", "tokens.cu", "ingest.cu", "contract.cu", "search.cu", "collective.cu", "capi.cu"]
CXX_SOURCES = ["solver.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the moeplace CUDA engine needs the CUDA 12.9 toolkit")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in CU_SOURCES + CXX_SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "moeplace_cuda.h"]
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False, defines=(), out: Path = None) -> Path:
    """Compile every kernel for sm_100a (-lineinfo) plus the host solver into one .so.
    ``defines``/``out`` build an experimental variant (e.g. MP_PF_AHEAD=0) next to the product lib."""
    global LIB
    product = LIB
    if out is not None:
        LIB = Path(out)
    try:
        return _build(force or out is not None, verbose, list(defines))
    finally:
        LIB = product


def _build(force: bool, verbose: bool, defines: list) -> Path:
    if not force and not _stale():
        return LIB
    nvcc = _nvcc()
    LIBDIR.mkdir(exist_ok=True)
    objdir = LIBDIR / ("obj" if not defines else "obj_" + "_".join(d.replace("=", "") for d in defines))
    objdir.mkdir(exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", str(ROOT / "include")]
    common += ["-D" + d for d in defines]
    objs = []
    jobs = []
    for src in CU_SOURCES:
        obj = objdir / (src + ".o")
        cmd = [nvcc, *ARCH, *common, "-Xptxas", "-v" if verbose else "-O3", "-c", str(CSRC / src), "-o", str(obj)]
        jobs.append((cmd, obj))
    for src in CXX_SOURCES:
        obj = objdir / (src + ".o")
        cmd = [nvcc, *common, "-Wno-deprecated-gpu-targets", "-x", "c++", "-c", str(CSRC / src), "-o", str(obj)]
        jobs.append((cmd, obj))
    procs = [(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True), cmd, obj)
             for cmd, obj in jobs]
    for p, cmd, obj in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed ({' '.join(cmd)}):\n{out}")
        if verbose and out:
            sys.stdout.write(out)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *objs, "-cudart", "static"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed ({' '.join(cmd)}):\n{r.stdout}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
