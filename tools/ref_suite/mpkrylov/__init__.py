"""``mpkrylov`` -> ``paper_2105_07544_b200`` drop-in shim (verification only).

Installs this repository's package under the reference's import name so the
reference's OWN test files (``/root/reference/pkg/tests``) run unmodified
against the B200 path: ``import mpkrylov as mk``, ``from mpkrylov.gmres
import gmres_cycle``, ``from mpkrylov.kernels import ...`` and
``python -m mpkrylov ...`` all resolve to the GPU implementation.  The
reference's ``model.py`` (SpMV traffic model) is out of scope and
is not aliased.  See ``tools/run_ref_suite.sh`` and INTEGRATION.md §2.
"""

import importlib
import os
import sys

_here = os.path.dirname(os.path.abspath(__file__))
_root = os.path.dirname(os.path.dirname(os.path.dirname(_here)))
if _root not in sys.path:
    sys.path.insert(0, _root)

import paper_2105_07544_b200 as _pkg  # noqa: E402

_SUBMODULES = ("errors", "gmres", "kernels", "mmio", "multiprecision", "precision",
               "preconditioners", "reorder", "sparse", "stencils", "cli")
for _name in _SUBMODULES:
    _mod = importlib.import_module("paper_2105_07544_b200." + _name)
    sys.modules["mpkrylov." + _name] = _mod
    globals()[_name] = _mod

from paper_2105_07544_b200 import *  # noqa: E402,F401,F403

__version__ = _pkg.__version__
__all__ = [n for n in dir(_pkg) if not n.startswith("_")]
