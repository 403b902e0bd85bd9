#!/bin/bash
# K1 in-step policy A/B: the new cluster rule vs the old one (OFB_K1_POLICY_OLD) vs split forced, all-resident steps
for M in new old split; do
  echo "== $M"
  case $M in new) E="";; old) E="OFB_K1_POLICY_OLD=1";; split) E="OFB_K1=split";; esac
  env $E timeout 900 python tools/small_step_probe.py --batches 1,2,4 --contexts 8192,16384,32768 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['shape'], d['B'], d['context'], round(d['us_per_layer'], 2))"
done
