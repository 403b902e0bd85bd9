# In-step K1 kernel / plan sweep with the late consumer wait (tools/k1_instep_sweep.py)
mkdir -p gpurun_out/k1instep
O=gpurun_out/k1instep
timeout 1500 python tools/k1_instep_sweep.py > $O/sweep.jsonl 2> $O/sweep.err; echo "sweep rc=$?"
