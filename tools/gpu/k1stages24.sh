#!/bin/bash
# K1 wide ring 24 stages: full variant sweep + bandwidth sweep + in-step probe (compare with r02_final2_* / r02_k1_variants_issue_loops.md)
mkdir -p gpurun_out/st24
timeout 1500 python tools/k1_variant_sweep.py > gpurun_out/st24/k1_variants.md 2> gpurun_out/st24/k1_variants.jsonl
timeout 600 python tools/k1_sweep.py > gpurun_out/st24/k1_sweep.md 2> /dev/null
timeout 900 python tools/small_step_probe.py --batches 1,2,4,8,16 --contexts 1024,4096,16384 > gpurun_out/st24/small_step.jsonl 2>&1
echo done
