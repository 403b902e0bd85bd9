# cfg3 host control under cProfile (live-wall), current code
mkdir -p gpurun_out/hostprof
timeout 900 python tools/cfg3_host_profile.py --requests 8 --top 60 > gpurun_out/hostprof/live_wall.txt 2>&1; echo "rc=$?"
