set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
free -g | head -2
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c1_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/c1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c1_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/c1_bench.json
timeout 900 python bench.py --config cfg4-serve --tp-emulate 8 > gpurun_out/c1_cfg4_tp8.json 2> gpurun_out/c1_cfg4_tp8.err; echo "cfg4 tp8 rc=$?"
tail -c 2000 gpurun_out/c1_cfg4_tp8.json; tail -20 gpurun_out/c1_cfg4_tp8.err
