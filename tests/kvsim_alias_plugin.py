"""pytest plugin: make ``import kvsim[.module]`` resolve to paper_2601_10729_b200.

Used by tests/test_reference_suite.py to run the reference's own unit tests
(/root/reference/pkg/tests, read in place, never copied) against this package.
"""

import importlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

_MODULES = ("core", "latency", "planner", "controller", "policies", "engine", "metrics",
            "workload", "defaults", "cli")


def _install_alias():
    pkg = importlib.import_module("paper_2601_10729_b200")
    sys.modules["kvsim"] = pkg
    for name in _MODULES:
        mod = importlib.import_module(f"paper_2601_10729_b200.{name}")
        sys.modules[f"kvsim.{name}"] = mod
        setattr(pkg, name, mod)


_install_alias()  # at plugin import: before the reference conftest imports kvsim
