"""Drop-in name for the reference package (``moeplace``, /root/reference/pkg/pyproject.toml:6).

Each ``moeplace.<module>`` IS the corresponding ``paper_2508_09229_b200.<module>`` object
(aliased in sys.modules), so classes and exceptions are identical whichever name a caller uses.
"""
import importlib
import sys

import paper_2508_09229_b200 as _impl

__version__ = _impl.__version__

for _name in _impl.MODULES:
    _mod = importlib.import_module(f"paper_2508_09229_b200.{_name}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
del _name, _mod
