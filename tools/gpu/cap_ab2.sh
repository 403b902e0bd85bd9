# A/B on one box: cap 256 everywhere (tools/gpu/head_lib) vs wide 256 / narrow 512 (current); K1 + executor GPU tests on the current library
mkdir -p gpurun_out/capab2
for i in 1 2; do
  OFB_LIB=tools/gpu/head_lib/liborbitflow_b200.so timeout 300 python tools/small_step_probe.py > gpurun_out/capab2/small_256_$i.jsonl 2>&1
  timeout 300 python tools/small_step_probe.py > gpurun_out/capab2/small_cur_$i.jsonl 2>&1
done
SWEEP_SHAPES=8B SWEEP_MODES=auto timeout 600 python tools/k1_instep_sweep.py --batches 1,2 --contexts 4096,40000,98304 > gpurun_out/capab2/long_cur.jsonl 2>&1
timeout 900 python -m pytest tests/test_executor_gpu.py tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -q -p no:cacheprovider > gpurun_out/capab2/tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/k1_sweep.py > gpurun_out/capab2/k1_sweep.md 2>&1; echo "sweep rc=$?"
