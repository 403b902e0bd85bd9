mkdir -p gpurun_out
for sp in 1 2 4; do
  for sh in "70B TP8" "70B TP4" "70B TP1"; do
    echo "splits=$sp"; OFB_K6_SPLITS=$sp timeout 120 python tools/oproj_bench.py --only "$sh" --no-emulated
  done
done > gpurun_out/c13_k6_splits.txt 2>&1
cat gpurun_out/c13_k6_splits.txt
