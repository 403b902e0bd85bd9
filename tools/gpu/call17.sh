mkdir -p gpurun_out
timeout 1500 python bench.py --config cfg3 > gpurun_out/c17_cfg3_40g.json 2> gpurun_out/c17_cfg3_40g.err; echo "cfg3 40g rc=$?"
tail -c 600 gpurun_out/c17_cfg3_40g.err
timeout 1500 python bench.py --config cfg3 --cfg3-budget-blocks 262144 > gpurun_out/c17_cfg3_16g.json 2> gpurun_out/c17_cfg3_16g.err; echo "cfg3 16g rc=$?"
tail -c 600 gpurun_out/c17_cfg3_16g.err
