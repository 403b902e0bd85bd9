timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_vllm_anchor_gpu.py tests/test_fullsize_gpu.py tests/test_torch_ops.py -x -q -p no:cacheprovider > gpurun_out/k1s2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/k1s2_pytest.log
timeout 600 python tools/k1_sweep.py > gpurun_out/k1_sweep_split2auto.md 2> gpurun_out/k1_sweep_split2auto.err; cat gpurun_out/k1_sweep_split2auto.md
timeout 300 python tools/small_step_probe.py
