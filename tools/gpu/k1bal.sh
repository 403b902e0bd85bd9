# In-step K1 split length vs SM balance (tools/k1_balance_sweep.py), auto and split pinned.
mkdir -p gpurun_out/k1bal
O=gpurun_out/k1bal
timeout 900 python tools/k1_balance_sweep.py > $O/auto.jsonl 2> $O/auto.err; echo "auto rc=$?"
OFB_K1=split timeout 900 python tools/k1_balance_sweep.py > $O/split.jsonl 2> $O/split.err; echo "split rc=$?"
