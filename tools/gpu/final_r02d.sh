# Final round-2 measurement pass on the committed code (after the late K1 wait, in-step policy, 512-block splits)
mkdir -p gpurun_out/final4
O=gpurun_out/final4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "gputest rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
for tp in 8 4 2 1; do
  timeout 1500 python bench.py --config cfg4-serve --tp-emulate $tp > $O/cfg4_serve_tp$tp.json 2> $O/cfg4_serve_tp$tp.err; echo "cfg4 tp$tp rc=$?"
done
timeout 2400 python bench.py --config cfg3 > $O/cfg3_40gib.json 2> $O/cfg3_40gib.err; echo "cfg3 rc=$?"
timeout 600 python tools/k1_sweep.py > $O/k1_sweep.md 2> $O/k1_sweep.err; echo "k1 sweep rc=$?"
timeout 300 python tools/small_step_probe.py > $O/small_step.jsonl 2>&1; echo "small rc=$?"
timeout 300 python tools/oproj_bench.py > $O/k6_oproj.jsonl 2>&1; echo "k6 rc=$?"
for c1 in k6 nccl; do timeout 600 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 6 --c1 $c1 > $O/decoder_probe_tp8_$c1.jsonl 2>&1; echo "probe $c1 rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"paged_gqa|kv_append|oproj|kv_prefill|attn_combine" --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_gqa_decode_kernel -s 2 -c 1 -o $O/k1split_cfg2layer -f python tools/attn_bench.py --batch 16 --hq 32 --hkv 8 --seq 32768 --layers 3 --iters 4 --variant split > /dev/null 2>&1; echo "ncu k1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oproj -s 30 -c 1 -o $O/k6_tp8 -f python tools/oproj_bench.py --only "70B TP8" --no-emulated > /dev/null 2>&1; echo "ncu k6 rc=$?"
