#!/bin/bash
# K1 after the issue-loop change and the refitted variant policy: parity, standalone sweep, in-step probe
timeout 1200 python -m pytest tests/test_kernels_gpu.py tests/test_executor_gpu.py tests/test_decoder_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
mkdir -p gpurun_out
timeout 1500 python tools/k1_variant_sweep.py > gpurun_out/k1_variants_policy.md 2>gpurun_out/k1_variants_policy.jsonl
cat gpurun_out/k1_variants_policy.md | cut -d'|' -f1-4,9-11
for M in new split; do
  echo "== in-step $M"
  case $M in new) E="";; split) E="OFB_K1=split";; esac
  env $E timeout 900 python tools/small_step_probe.py --batches 1,2,4,8,16 --contexts 1024,4096,8192,16384 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['shape'], d['B'], d['context'], round(d['us_per_layer'], 2))" | tee gpurun_out/k1_instep_$M.txt
done
