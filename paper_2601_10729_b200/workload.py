"""Synthetic request traces and the canonical trace file format.

Out of the data path (reuse unchanged): this is the
reference's own module (/root/reference/pkg/src/kvsim/workload.py:1-178), executed unmodified by
``_kvsim.load`` with its relative imports bound to this package.
The config-3 mixed-length trace of BASELINE.json is this generator's
output for seed 3.
"""

from ._kvsim import reexport as _reexport

__all__ = _reexport("workload", globals())
