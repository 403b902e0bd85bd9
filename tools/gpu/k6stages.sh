#!/bin/bash
# K6 ring depth when a CTA's whole K range fits the ring (TP8 o-proj: 8 chunks per CTA): stage cap sweep
for ST in 8 7 6 5 4; do
  echo "== stages $ST"
  for rep in 1 2; do
  OFB_K6_STAGES=$ST timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    if d['shape'] in ('70B TP8', '8B TP4 B16', '70B TP8 qkv'): print(d['shape'], round(d['k6_us'], 2), round(d['cublas_us'], 2))"
  done
done
