# A/B: the previous library (tools/gpu/head_lib) vs the current one (OFB_K6_MC=0 unless set), same box
fmt='import sys,json
for l in sys.stdin:
  try: d=json.loads(l); print(d["shape"], round(d["k6_us"],2), round(d["cublas_us"],2))
  except Exception: pass'
for i in 1 2; do
  echo "== head lib"; OFB_LIB=tools/gpu/head_lib/liborbitflow_b200.so timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | python -c "$fmt"
  echo "== current"; OFB_K6_MC=${MC:-0} timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | python -c "$fmt"
done
echo "== decoder head"; OFB_LIB=tools/gpu/head_lib/liborbitflow_b200.so timeout 300 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 5 2>&1 | tail -1 | cut -c80-200
echo "== decoder current"; OFB_K6_MC=${MC:-0} timeout 300 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 5 2>&1 | tail -1 | cut -c80-200
