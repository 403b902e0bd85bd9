#!/bin/bash
# K6 split-K reduce-scatter (OFB_K6_RS=1, default) vs the leader reduction (OFB_K6_RS=0): parity, sanitizers, bench, decoder
timeout 900 python -m pytest tests/test_oproj_gpu.py tests/test_decoder_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for shape in "32 8192 1280" "32 1024 8192" "19 4096 1280" "16 1024 4096"; do
  for t in synccheck racecheck memcheck; do r=$(timeout 600 compute-sanitizer --tool $t python tools/k6_sync_case.py $shape 2>&1 | grep -E "SUMMARY" | head -1); echo "$shape $t: $r"; done
done
for R in 0 1 0 1; do
  echo "== rs $R"
  OFB_K6_RS=$R timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | grep "^{" | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['shape'], round(d['k6_us'], 2), round(d['cublas_us'], 2), round(d['max_abs_err_vs_fp32'], 4))"
done
for R in 0 1; do OFB_K6_RS=$R timeout 600 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 6 --c1 k6 2>&1 | grep step_ms | cut -c1-160; done
