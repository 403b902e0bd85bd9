#!/bin/bash
# K1 with converged producer warps / incremental ring counters: parity, the full variant sweep, in-step probe per variant
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
mkdir -p gpurun_out
timeout 1500 python tools/k1_variant_sweep.py > gpurun_out/k1_variants_elect.md 2>gpurun_out/k1_variants_elect.jsonl
cat gpurun_out/k1_variants_elect.md
for V in split cluster; do echo "== in-step $V"; OFB_K1=$V timeout 900 python tools/small_step_probe.py 2>&1 | tail -8; done
echo "== in-step auto"; timeout 900 python tools/small_step_probe.py 2>&1 | tail -8
