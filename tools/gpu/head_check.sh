# Session re-entry check on HEAD: GPU suite, default bench, K6 vs cuBLAS, small-step probe.
mkdir -p gpurun_out/head
O=gpurun_out/head
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "gputest rc=$?"
timeout 600 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench rc=$?"
timeout 300 python tools/oproj_bench.py > $O/k6_oproj.jsonl 2>&1; echo "k6 rc=$?"
timeout 300 python tools/small_step_probe.py > $O/small_step.jsonl 2>&1; echo "small rc=$?"
timeout 600 python tools/k1_sweep.py > $O/k1_sweep.md 2> $O/k1_sweep.err; echo "k1 sweep rc=$?"
