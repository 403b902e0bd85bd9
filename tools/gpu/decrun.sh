# whole-decoder TP8 step A/B (current vs HEAD library) + decoder / executor tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_executor_gpu.py tests/test_kernels_gpu.py -x -q -p no:cacheprovider > gpurun_out/dec_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/dec_pytest.log
for p in 4088 65528; do
  echo "== new prompt=$p"; timeout 600 python tools/decoder_probe.py --tp 8 --prompt $p --steps 6 2>&1 | tail -1
  echo "== head prompt=$p"; OFB_LIB=tools/gpu/head_lib/liborbitflow_b200.so timeout 600 python tools/decoder_probe.py --tp 8 --prompt $p --steps 6 2>&1 | tail -1
done
timeout 300 python tools/small_step_probe.py
