mkdir -p gpurun_out/tin
timeout 900 python -m pytest tests/test_executor_gpu.py -q -p no:cacheprovider -k "attention_only" > gpurun_out/tin/log.txt 2>&1; echo "rc=$?"
