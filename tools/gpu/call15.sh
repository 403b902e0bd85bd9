mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_oproj_gpu.py -x -q -p no:cacheprovider > gpurun_out/c15_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/c15_pytest.log
for sp in 1 2 4; do echo "splits=$sp"; OFB_K6_SPLITS=$sp timeout 120 python tools/oproj_bench.py --no-emulated; done > gpurun_out/c15_k6.txt 2>&1
for sp in 2; do echo "splits=$sp"; OFB_K6_SPLITS=$sp timeout 120 python tools/k6_trace.py 32 1024 8192; done >> gpurun_out/c15_k6.txt 2>&1
