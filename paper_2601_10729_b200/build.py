"""Build recipe for the sm_100a data-path library (``liborbitflow_b200.so``).

Plain nvcc, in-tree output (``paper_2601_10729_b200/_lib``) so the built
library travels with the repo snapshot to the GPU box.  No torch extension
machinery: the library exposes the C ABI declared in
``include/orbitflow_b200.h`` and is bound with ctypes (``_native.py``).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB_NAME = "liborbitflow_b200.so"
SOURCES = ["decode_attention.cu", "decode_attention_stream.cu", "decode_attention_cluster.cu", "kv_append.cu", "kv_prefill.cu", "runtime.cu",
           "oproj_allreduce.cu", "decoder_glue.cu", "planner_gpu.cu",
           "planner.cpp"]

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
    "-Xcompiler", "-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-cudart", "shared",
]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found: the sm_100a library cannot be built")
    return cand


def lib_path() -> Path:
    return OUT_DIR / LIB_NAME


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_verbose: bool = False) -> Path:
    """Compile every .cu into one shared library; returns its path."""
    OUT_DIR.mkdir(exist_ok=True)
    target = lib_path()
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "orbitflow_b200.h"]
    if not force and not _stale(target, deps):
        return target
    objs = []
    for src in SOURCES:
        obj = OUT_DIR / (Path(src).stem + ".o")
        cmd = [nvcc(), *ARCH_FLAGS, *NVCC_FLAGS, "-I", str(ROOT / "include"), "-c", str(CSRC / src), "-o", str(obj)]
        cmd.extend(["-Xcompiler", "-fvisibility=hidden"])
        if src.endswith(".cpp"):   # host-only planner: no FMA contraction (bit-exact plans)
            cmd.extend(["-x", "c++", "-Xcompiler", "-ffp-contract=off", "-Xcompiler", "-pthread"])
        if ptxas_verbose:
            cmd.extend(["-Xptxas", "-v"])
        _run(cmd, verbose or ptxas_verbose)
        objs.append(str(obj))
    tmp = target.with_suffix(".so.tmp")
    _run([nvcc(), *ARCH_FLAGS, "-shared", "-cudart", "shared", "-Xcompiler", "-pthread", "-o", str(tmp), *objs, "-lcuda"
          if _has_libcuda() else "-L/usr/local/cuda/lib64/stubs"], verbose)
    os.replace(tmp, target)
    return target


TORCH_OPS_NAME = "liborbit_torch_ops.so"


def torch_ops_path() -> Path:
    return OUT_DIR / TORCH_OPS_NAME


def build_torch_ops(verbose: bool = False, force: bool = False) -> Path:
    """The ``orbit::`` torch.library registration (csrc/torch_ops.cpp): host-only
    C++ against torch's headers, linked to liborbitflow_b200.so (found next to it
    through $ORIGIN), so ``torch.ops.orbit.*`` and the ctypes binding call the same
    kernels.  Plain g++ - no JIT cache, the .so stays in-tree and travels."""
    from torch.utils import cpp_extension

    lib = build(verbose=verbose)
    target = torch_ops_path()
    src = CSRC / "torch_ops.cpp"
    if not force and not _stale(target, [src, lib, ROOT / "include" / "orbitflow_b200.h"]):
        return target
    import torch

    incs = [f"-I{p}" for p in cpp_extension.include_paths(device_type="cuda")]
    libdirs = cpp_extension.library_paths(device_type="cuda")
    abi = int(torch._C._GLIBCXX_USE_CXX11_ABI)
    tmp = target.with_suffix(".so.tmp")
    cmd = [os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-shared", "-fPIC",
           f"-D_GLIBCXX_USE_CXX11_ABI={abi}", "-DTORCH_EXTENSION_NAME=orbit_torch_ops",
           f"-I{ROOT / 'include'}", *incs, str(src), "-o", str(tmp),
           f"-L{OUT_DIR}", "-l:" + LIB_NAME, "-Wl,-rpath,$ORIGIN",
           *[f"-L{d}" for d in libdirs], "-lc10", "-lc10_cuda", "-ltorch_cpu", "-ltorch_cuda",
           "-ltorch", "-ltorch_python"]
    _run(cmd, verbose)
    os.replace(tmp, target)
    return target


REFERENCE_SRC = Path("/root/reference/pkg")
REFERENCE_TARGET = ROOT / "baseline" / "_ref"


def install_reference(force: bool = False) -> Path | None:
    """Install the unmodified reference ``kvsim`` into ``baseline/_ref`` (offline).

    The engine and the out-of-scope harness modules execute the reference's own
    sources (``_kvsim.py``); ``baseline/_ref`` is git-ignored but travels to the
    GPU box with the repo snapshot.  Installed from a scratch copy because the
    reference tree is read-only.  Returns the package directory, or None when
    the reference tree is absent (GPU box: the snapshot already carries it).
    """
    pkg = REFERENCE_TARGET / "kvsim"
    if (pkg / "engine.py").is_file() and not force:
        return pkg
    if not (REFERENCE_SRC / "pyproject.toml").is_file():
        return None
    import tempfile

    with tempfile.TemporaryDirectory() as tmp:
        src = Path(tmp) / "pkg"
        shutil.copytree(REFERENCE_SRC, src)
        _run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
              "--no-deps", "--find-links", "/opt/wheelhouse", "--upgrade", "--target",
              str(REFERENCE_TARGET), str(src)], False)
    return pkg


def _has_libcuda() -> bool:
    return False  # the driver entry point is resolved at run time (cudaGetDriverEntryPoint)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose and res.stderr:
        print(res.stderr, file=sys.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"build step failed ({res.returncode}):\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")


if __name__ == "__main__":
    p = build(verbose="-v" in sys.argv, force="-f" in sys.argv, ptxas_verbose="--ptxas" in sys.argv)
    print(p)
