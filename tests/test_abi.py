"""The C-ABI library builds, loads and exports exactly what include/*.h declares.

CPU-only: no compute calls (there is no GPU in the build container)."""

import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "orbitflow_b200.h").read_text()
    return sorted(set(re.findall(r"OFB_API[^;(]*?\b(ofb_\w+)\s*\(", text, re.S)))


def test_header_declares_the_boundary():
    names = _declared()
    for want in ("ofb_decode_attention", "ofb_kv_append", "ofb_runtime_decode_step",
                 "ofb_runtime_migrate", "ofb_host_alloc"):
        assert want in names


def test_library_exports_every_declared_symbol():
    from paper_2601_10729_b200 import _native, build

    path = build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", str(path)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (ofb_\w+)", out))
    assert set(_declared()) <= exported
    assert set(_native.SIGNATURES) == set(_declared())


def test_library_loads_and_binds():
    from paper_2601_10729_b200 import _native

    lib = _native.load()
    assert lib.ofb_version().decode().startswith("orbitflow-b200")
    # workspace sizing is host arithmetic, safe without a GPU
    assert lib.ofb_attention_workspace_bytes(16, 32, 8, 32768) > 0


def test_sm100a_sass_present():
    from paper_2601_10729_b200 import build

    path = build.build()
    sass = subprocess.run(["cuobjdump", "-sass", str(path)], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass          # TMA tile loads
    assert "HMMA" in sass             # tensor-core tiles of the GQA group
    assert "LDSM" in sass
