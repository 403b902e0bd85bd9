mkdir -p gpurun_out/wall
timeout 1200 python tools/cfg3_wall_probe.py > gpurun_out/wall/probe.jsonl 2> gpurun_out/wall/probe.err; echo "rc=$?"
