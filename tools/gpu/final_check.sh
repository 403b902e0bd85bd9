# Last check on the committed code: full GPU suite, smoke, default bench
mkdir -p gpurun_out/fcheck
O=gpurun_out/fcheck
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gputest.log 2>&1; echo "gputest rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; echo "bench rc=$?"
timeout 300 python tools/small_step_probe.py > $O/small_step.jsonl 2>&1; echo "small rc=$?"
