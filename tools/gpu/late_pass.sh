# Measurement pass after the K1 late wait / in-step policy: GPU suite, default bench, cfg4-serve TP8/TP4,
# small-step probe, K1 sweep (standalone), launch list + ncu full of K1 (cfg2 layer)
mkdir -p gpurun_out/late
O=gpurun_out/late
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "gputest rc=$?"
timeout 600 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench rc=$?"
for tp in 8 4; do
  timeout 1500 python bench.py --config cfg4-serve --tp-emulate $tp > $O/cfg4_serve_tp$tp.json 2> $O/cfg4_serve_tp$tp.err; echo "cfg4 tp$tp rc=$?"
done
timeout 300 python tools/small_step_probe.py > $O/small_step.jsonl 2>&1; echo "small rc=$?"
timeout 600 python tools/k1_sweep.py > $O/k1_sweep.md 2> $O/k1_sweep.err; echo "k1 sweep rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"paged_gqa|kv_append|oproj|kv_prefill|attn_combine" --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_gqa_decode_kernel -s 2 -c 1 -o $O/k1split_cfg2layer -f python tools/attn_bench.py --batch 16 --hq 32 --hkv 8 --seq 32768 --layers 3 --iters 4 --variant split > /dev/null 2>&1; echo "ncu k1 rc=$?"
