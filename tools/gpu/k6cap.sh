fmt='import sys,json
for l in sys.stdin:
  try: d=json.loads(l); print(d["shape"], round(d["k6_us"],2), round(d["cublas_us"],2), round(d["speedup_vs_cublas"],3))
  except Exception: print(l.strip()[:300])'
for cap in 4 8; do echo "== cap $cap"; OFB_K6_SPLIT_CAP=$cap timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | python -c "$fmt"; done
OFB_K6_SPLIT_CAP=8 timeout 300 python -m pytest tests/test_oproj_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
