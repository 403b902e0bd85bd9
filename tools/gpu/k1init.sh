#!/bin/bash
# K1 parallel ring-barrier init (+ 24-stage wide ring): parity, sanitizers, latency sweep, in-step probe
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_executor_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for t in synccheck racecheck; do r=$(timeout 900 compute-sanitizer --tool $t python tools/sanitize_case.py 2>&1 | grep -E "SUMMARY" | head -1); echo "$t: $r"; done
mkdir -p gpurun_out/init
timeout 1500 python tools/k1_variant_sweep.py --quick > gpurun_out/init/k1_variants.md 2> gpurun_out/init/k1_variants.jsonl
timeout 900 python tools/small_step_probe.py --batches 1,2,4,8,16 --contexts 1024,4096,16384 > gpurun_out/init/small_step.jsonl 2>&1
echo done
