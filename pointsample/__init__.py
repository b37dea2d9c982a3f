"""Import alias: the reference package name (pkg/pyproject.toml:6,
``pointsample``) for the B200 implementation in ``paper_2507_23480_b200``.

``import pointsample._kernels`` / ``from pointsample import core, mdps`` give
the B200 modules themselves (the same module objects), so a reference
orchestrator swaps implementations by putting this repo first on sys.path.
"""

import importlib
import sys

_IMPL = "paper_2507_23480_b200"
_MODULES = ("core", "_kernels", "baselines", "curve", "mdps", "neighbors", "quality", "harness", "engine",
            "pointsplit")

for _m in _MODULES:
    _mod = importlib.import_module(f"{_IMPL}.{_m}")
    sys.modules[f"{__name__}.{_m}"] = _mod
    globals()[_m] = _mod

del _m, _mod
