# K1 latency-bound A/B: kernel parity tests, variant sweep (quick) for current and HEAD libraries, traces
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_vllm_anchor_gpu.py -x -q -p no:cacheprovider > gpurun_out/k1_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/k1_pytest.log
echo "== new"; timeout 600 python tools/k1_variant_sweep.py --quick 2> gpurun_out/k1_var_new.jsonl | tee gpurun_out/k1_var_new.md
echo "== head"; OFB_LIB=tools/gpu/head_lib/liborbitflow_b200.so timeout 600 python tools/k1_variant_sweep.py --quick 2> gpurun_out/k1_var_head.jsonl | tee gpurun_out/k1_var_head.md
python tools/k1_split_trace.py --batch 1 --hq 32 --hkv 8 --seq 4096 > gpurun_out/k1_tr_8b.json
python tools/k1_split_trace.py --batch 1 --hq 8 --hkv 1 --seq 16384 > gpurun_out/k1_tr_tp8.json
python tools/k1_split_trace.py --batch 1 --hq 8 --hkv 1 --seq 16384 --variant cluster > gpurun_out/k1_tr_tp8_cluster.json
