"""Re-export of the synthetic workload generator (``workloads``), which lives
outside the product package so that generating inputs never loads
libgnetmon.so (bench.py's reference arm)."""
import os as _os
import sys as _sys

_root = _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))
if _root not in _sys.path:
    _sys.path.insert(0, _root)

from workloads import *  # noqa: E402,F401,F403
from workloads import _lib, _Spec  # noqa: E402,F401
