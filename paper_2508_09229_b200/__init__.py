"""B200-native engine for the data-parallel core of arXiv 2508.09229 (topology-aware MoE expert
placement), exposed with the reference package's API: ``import moeplace`` resolves to the
modules below (see moeplace/__init__.py).

Modules mirror SPEC.md: ``topology``, ``model_trace``, ``placement``, ``solver``, ``eval``,
``cli`` and ``errors``.  The hot path runs in hand-written sm_100a CUDA kernels behind the C-ABI
in ``include/moeplace_cuda.h`` (library ``lib/libmoeplace_cuda.so``, bound in ``_lib``).
"""

__version__ = "0.1.0"

from . import errors  # noqa: F401  (import order: errors first, no torch needed)

MODULES = ("errors", "topology", "model_trace", "placement", "solver", "eval", "cli", "search", "shard")
