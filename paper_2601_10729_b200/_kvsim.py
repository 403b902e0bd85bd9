"""Load modules of the installed reference ``kvsim`` unmodified, bound to this package.

The serving loop (``engine``) and the out-of-scope harness around the data path
(``metrics``, ``workload``, ``defaults``, ``policies``, ``cli``) are the
reference's own code, not restatements: SURVEY.md section 2 says to reuse them
unchanged.  Each module's source file is executed as a private submodule of
this package (``paper_2601_10729_b200._ref_<name>``), so its relative imports
(``from .planner import solve`` ...) bind to this package's restated host
modules - the native exact planner included - and this package adds only the
executor seam on top (``engine.Simulation``).

Where the reference lives (first hit wins):
  1. ``$OFB_KVSIM_SRC`` (a directory holding ``engine.py`` etc.);
  2. ``<repo>/baseline/_ref/kvsim`` - the one offline install the task allows
     (``python -m pip install --no-index --target baseline/_ref <reference>``;
     ``build.install_reference()`` runs it);
  3. ``/root/reference/pkg/src/kvsim`` (the read-only reference tree).
A missing reference raises ``ImportError`` naming these places.
"""

from __future__ import annotations

import importlib.util
import os
import sys
from pathlib import Path

_PKG = __name__.rsplit(".", 1)[0]
_ROOT = Path(__file__).resolve().parent.parent
_CANDIDATES = (
    _ROOT / "baseline" / "_ref" / "kvsim",
    Path("/root/reference/pkg/src/kvsim"),
)


def source_dir() -> Path:
    env = os.environ.get("OFB_KVSIM_SRC")
    dirs = ([Path(env)] if env else []) + list(_CANDIDATES)
    for d in dirs:
        if (d / "engine.py").is_file():
            return d
    raise ImportError(
        "the reference kvsim sources were not found (looked in $OFB_KVSIM_SRC, "
        f"{', '.join(str(d) for d in _CANDIDATES)}); install them with "
        "`python -c 'from paper_2601_10729_b200 import build; build.install_reference()'`")


def load(name: str):
    """The reference module ``kvsim.<name>``, executed with this package as its parent."""
    full = f"{_PKG}._ref_{name}"
    mod = sys.modules.get(full)
    if mod is not None:
        return mod
    path = source_dir() / f"{name}.py"
    spec = importlib.util.spec_from_file_location(full, path)
    mod = importlib.util.module_from_spec(spec)
    mod.__package__ = _PKG          # relative imports resolve inside this package
    sys.modules[full] = mod
    try:
        spec.loader.exec_module(mod)
    except BaseException:
        sys.modules.pop(full, None)
        raise
    return mod


def reexport(name: str, namespace: dict) -> list[str]:
    """Bind every public name of reference module ``name`` into ``namespace``."""
    mod = load(name)
    names = [k for k in vars(mod) if not k.startswith("__")]
    for k in names:
        namespace.setdefault(k, getattr(mod, k))
    return [k for k in names if not k.startswith("_")]
