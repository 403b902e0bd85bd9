# cluster K1 with a shallower ring (more clusters per wave) vs split, latency-bound 8B / 70B shapes
for st in 24 12 8; do
  echo "== stages $st"
  for v in cluster split; do
    OFB_K1=$v OFB_K1_CLUSTER_STAGES=$st timeout 300 python tools/small_step_probe.py | python -c "import sys,json
for l in sys.stdin:
  d=json.loads(l); print('$v', d['shape'], d['B'], d['context'], round(d['us_per_layer'],2))"
  done
done
