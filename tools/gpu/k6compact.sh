#!/bin/bash
# K6 epilogues rolled over 8-column TMEM loads (+ reduce-scatter at 8 splits): parity, sanitizers, bench, decoder, trace
timeout 900 python -m pytest tests/test_oproj_gpu.py tests/test_decoder_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for shape in "32 8192 1280" "32 1024 8192" "19 4096 1280" "200 1024 2048"; do
  for t in synccheck racecheck memcheck; do r=$(timeout 600 compute-sanitizer --tool $t python tools/k6_sync_case.py $shape 2>&1 | grep -E "SUMMARY" | head -1); echo "$shape $t: $r"; done
done
for rep in 1 2; do
  timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | grep "^{" | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['shape'], round(d['k6_us'], 2), round(d['cublas_us'], 2), round(d['max_abs_err_vs_fp32'], 4))"
done
for i in 1 2; do timeout 600 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 6 --c1 k6 2>&1 | grep step_ms | cut -c1-160; done
timeout 300 python tools/k6_trace.py 32 1024 8192 2>&1 | tail -1
timeout 300 python tools/k6_trace.py 32 8192 1280 2>&1 | tail -1
