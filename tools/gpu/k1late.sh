# K1 split: consumers' PDL wait moved after the split's math in attention-only steps (OFB_K1_LATE=1), wide / narrow
mkdir -p gpurun_out/k1late
O=gpurun_out/k1late
for late in 0 1; do for wide in auto 0; do
  if [ $wide = auto ]; then W=""; else W="OFB_K1_WIDE=$wide"; fi
  env OFB_K1=split OFB_K1_LATE=$late $W timeout 900 python tools/k1_balance_sweep.py --batches 1,2 > $O/late${late}_wide${wide}.jsonl 2> $O/late${late}_wide${wide}.err; echo "late=$late wide=$wide rc=$?"
done; done
OFB_K1_LATE=1 timeout 600 python tools/small_step_probe.py > $O/small_late1.jsonl 2>&1; echo "small rc=$?"
OFB_K1_LATE=1 timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "executor or fullsize or kernels or step" > $O/gputest_late1.log 2>&1; echo "tests rc=$?"
