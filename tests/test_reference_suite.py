"""Run the reference's own test suite (170 tests) against this package.

The reference tests are executed in place from /root/reference (never copied
into this repo) with ``kvsim`` aliased to ``paper_2601_10729_b200``.  This pins
the host API - placement plans, deferral decisions, block tables, the
transfer-schedule oracle equivalence, the golden Fig.-3 numbers - to the
reference's own assertions.  Skipped where /root/reference is absent (the GPU
box); the committed golden fixtures (tests/golden) cover that side.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

REF_TESTS = Path("/root/reference/pkg/tests")
HERE = Path(__file__).resolve().parent


@pytest.mark.skipif(not REF_TESTS.exists(), reason="reference tree not mounted")
def test_reference_suite_passes_against_b200_package(tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(HERE), str(REF_TESTS), str(HERE.parent)])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p",
           "kvsim_alias_plugin", "--rootdir", str(tmp_path), "-c", os.devnull, str(REF_TESTS)]
    res = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=900)
    tail = "\n".join(res.stdout.splitlines()[-30:])
    assert res.returncode == 0, f"reference suite failed against this package:\n{tail}\n{res.stderr[-2000:]}"
    assert " passed" in tail and "failed" not in tail
