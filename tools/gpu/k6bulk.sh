#!/bin/bash
# K6 split-K partials by one DSMEM bulk copy + mbarrier (OFB_K6_BULK=1) vs per-thread DSMEM stores + cluster barrier
OFB_K6_BULK=1 timeout 900 python -m pytest tests/test_oproj_gpu.py tests/test_decoder_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for t in synccheck racecheck memcheck; do r=$(OFB_K6_BULK=1 timeout 600 compute-sanitizer --tool $t python tools/k6_sync_case.py 32 8192 1280 2>&1 | grep -E "SUMMARY" | head -1); echo "$t: $r"; done
for B in 0 1 0 1; do
  echo "== bulk $B"
  OFB_K6_BULK=$B timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | grep "^{" | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['shape'], round(d['k6_us'], 2), round(d['cublas_us'], 2))"
done
for B in 0 1; do OFB_K6_BULK=$B timeout 600 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 6 --c1 k6 2>&1 | grep step_ms | cut -c1-160; done
