# In-step policy with the late wait + balanced plan: sweep (auto should track the best), small-step probe, GPU suite, cfg3
mkdir -p gpurun_out/k1p2
O=gpurun_out/k1p2
timeout 1500 python tools/k1_instep_sweep.py > $O/sweep.jsonl 2> $O/sweep.err; echo "sweep rc=$?"
timeout 300 python tools/small_step_probe.py > $O/small_step.jsonl 2>&1; echo "small rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "gputest rc=$?"
timeout 2400 python bench.py --config cfg3 > $O/cfg3_40gib.json 2> $O/cfg3_40gib.err; echo "cfg3 rc=$?"
