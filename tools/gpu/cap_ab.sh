# A/B on one box: split block-table run cap 256 (tools/gpu/head_lib) vs 512 (current), small-step probe + long in-step shapes, twice each
mkdir -p gpurun_out/capab
for i in 1 2; do
  OFB_LIB=tools/gpu/head_lib/liborbitflow_b200.so timeout 300 python tools/small_step_probe.py > gpurun_out/capab/small_256_$i.jsonl 2>&1
  timeout 300 python tools/small_step_probe.py > gpurun_out/capab/small_512_$i.jsonl 2>&1
done
SWEEP_SHAPES=8B SWEEP_MODES=auto OFB_LIB=tools/gpu/head_lib/liborbitflow_b200.so timeout 600 python tools/k1_instep_sweep.py --batches 1,2 --contexts 4096,40000,98304 > gpurun_out/capab/long_256.jsonl 2>&1
SWEEP_SHAPES=8B SWEEP_MODES=auto timeout 600 python tools/k1_instep_sweep.py --batches 1,2 --contexts 4096,40000,98304 > gpurun_out/capab/long_512.jsonl 2>&1
echo done
