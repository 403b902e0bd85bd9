# Balanced in-step plan past 256 blocks per split (cfg3's long requests), parity tests, cfg3
mkdir -p gpurun_out/k1long
O=gpurun_out/k1long
SWEEP_SHAPES=8B SWEEP_MODES=auto,split,bal timeout 1200 python tools/k1_instep_sweep.py --batches 1,2,3 --contexts 24576,40000,65536,98304,131072 --max-tokens 262144 > $O/sweep.jsonl 2> $O/sweep.err; echo "sweep rc=$?"
timeout 900 python -m pytest tests/test_executor_gpu.py tests/test_kernels_gpu.py -q -p no:cacheprovider > $O/tests.log 2>&1; echo "tests rc=$?"
timeout 2400 python bench.py --config cfg3 > $O/cfg3_40gib.json 2> $O/cfg3_40gib.err; echo "cfg3 rc=$?"
