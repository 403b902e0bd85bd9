#!/bin/bash
# K1 split length that fills the SMs (18 splits x 8 KV heads = 144 CTAs) vs the power-of-two pick, 8B B=1 in a step
run() { OFB_K1_BPS=$3 timeout 300 python tools/small_step_probe.py --batches $1 --contexts $2 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    if d['shape'] == '8B': print(d['shape'], d['B'], d['context'], 'bps', '$3', round(d['us_per_layer'], 2))"; }
for cfg in "1 8192 32" "1 8192 29" "1 16384 64" "1 16384 57" "1 32768 128" "1 32768 114" "1 65536 256" "1 65536 228" "2 16384 64" "2 16384 114"; do
  set -- $cfg; run $1 $2 $3
done
