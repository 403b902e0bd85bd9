mkdir -p gpurun_out
for sp in 1 2; do echo "splits=$sp"; OFB_K6_SPLITS=$sp timeout 120 python tools/k6_trace.py 32 1024 8192; OFB_K6_SPLITS=$sp timeout 120 python tools/k6_trace.py 32 3584 8192; done > gpurun_out/c14_k6_trace.txt 2>&1
cat gpurun_out/c14_k6_trace.txt
