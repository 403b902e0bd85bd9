# K6: two CTAs per SM (ring <= 4 stages) with an early launch_dependents vs the default
for CFG in "8 0" "8 1" "4 0" "4 1" "3 1"; do set -- $CFG
  echo "== stages $1 early $2"
  OFB_K6_STAGES=$1 OFB_K6_EARLY=$2 timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['shape'], round(d['k6_us'], 2), round(d['cublas_us'], 2))"
done
