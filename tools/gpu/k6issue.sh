#!/bin/bash
# K6 with the converged-warp issue loops: parity, sanitizers, the projection shapes.
timeout 900 python -m pytest tests/test_oproj_gpu.py tests/test_decoder_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
for shape in "32 1024 8192" "32 8192 1280" "19 4096 1280" "32 8192 8192"; do
  for t in synccheck racecheck memcheck; do
    r=$(timeout 300 compute-sanitizer --tool $t python tools/k6_sync_case.py $shape 2>&1 | grep -E "SUMMARY" | head -1)
    echo "$shape $t: $r"
  done
done
for rep in 1 2; do
  timeout 300 python tools/oproj_bench.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d.get('shape', d.get('name')), round(d.get('k6_us', 0), 2), round(d.get('cublas_us', 0), 2))"
done
