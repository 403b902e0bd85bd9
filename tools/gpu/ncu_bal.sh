# ncu --set full of one in-step K1 launch on the balanced narrow plan (8B, B=1, 16K) and one on the cost-model plan
mkdir -p gpurun_out/ncubal
SWEEP_SHAPES=8B SWEEP_MODES=bal timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_gqa_decode -s 100 -c 1 -o gpurun_out/ncubal/k1_bal_8b_b1_16k -f python tools/k1_instep_sweep.py --batches 1 --contexts 16384 > gpurun_out/ncubal/bal.log 2>&1; echo "bal rc=$?"
SWEEP_SHAPES=8B SWEEP_MODES=split timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_gqa_decode -s 100 -c 1 -o gpurun_out/ncubal/k1_split_8b_b1_16k -f python tools/k1_instep_sweep.py --batches 1 --contexts 16384 > gpurun_out/ncubal/split.log 2>&1; echo "split rc=$?"
