# K6 A/B: tests, chain bench (current vs HEAD library), per-CTA trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_oproj_gpu.py -x -q -p no:cacheprovider > gpurun_out/k6_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/k6_pytest.log
fmt='import sys,json
for l in sys.stdin:
  try: d=json.loads(l); print(d["shape"], round(d["k6_us"],2), round(d["cublas_us"],2), round(d["speedup_vs_cublas"],3))
  except Exception: print(l.strip()[:300])'
for rep in 1 2; do
echo "== new"; timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | tee gpurun_out/k6_new.jsonl | python -c "$fmt"
echo "== head"; OFB_LIB=tools/gpu/head_lib/liborbitflow_b200.so timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | tee gpurun_out/k6_head.jsonl | python -c "$fmt"
done
timeout 100 python tools/k6_trace.py
