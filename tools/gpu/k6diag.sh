# K6 issue-loop A/B: stream only (diag 1), + MMAs (diag 2), full (0), ring depth 8 / 6
timeout 600 python -m pytest tests/test_oproj_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for ST in 8 6; do for D in 0 2 1; do
  echo "== stages $ST diag $D"
  OFB_K6_STAGES=$ST OFB_K6_DIAG=$D timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['shape'], round(d['k6_us'], 2), round(d['cublas_us'], 2))"
done; done
