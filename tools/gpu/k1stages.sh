#!/bin/bash
# K1 wide split kernel ring depth A/B (build-time constant): the cfg3-regime in-step probe + latency sweep
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 900 python tools/small_step_probe.py --batches 1,2,4 --contexts 8192,16384,32768 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['shape'], d['B'], d['context'], round(d['us_per_layer'], 2))"
