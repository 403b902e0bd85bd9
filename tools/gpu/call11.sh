mkdir -p gpurun_out
timeout 300 ncu --section SourceCounters --section WarpStateStats --import-source on --clock-control none --warp-sampling-interval 0 -k regex:paged_gqa_decode_cluster --launch-skip 4 -c 1 -o gpurun_out/c11_cluster -f python tools/k1_split_trace.py --variant cluster --batch 1 --hq 8 --hkv 1 --seq 16384 > gpurun_out/c11_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/c11_ncu.log
