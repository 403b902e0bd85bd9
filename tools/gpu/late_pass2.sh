# Second pass on the late-wait code: smoke, reference arm (with host DRAM bandwidth), cfg3 again, decoder probe both arms, K6 vs cuBLAS
mkdir -p gpurun_out/late2
O=gpurun_out/late2
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
timeout 2400 python bench.py --config cfg3 > $O/cfg3_40gib.json 2> $O/cfg3_40gib.err; echo "cfg3 rc=$?"
for c1 in k6 nccl; do timeout 600 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 6 --c1 $c1 > $O/decoder_probe_tp8_$c1.jsonl 2>&1; echo "probe $c1 rc=$?"; done
timeout 300 python tools/oproj_bench.py > $O/k6_oproj.jsonl 2>&1; echo "k6 rc=$?"
