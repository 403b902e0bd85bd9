mkdir -p gpurun_out
timeout 300 ncu --set full --import-source on --clock-control none -k regex:paged_gqa_decode_kernel --launch-skip 4 -c 1 -o gpurun_out/c6_split_tp8_b1_16k -f python tools/k1_split_trace.py --batch 1 --hq 8 --hkv 1 --seq 16384 > gpurun_out/c6_ncu_split.log 2>&1; echo "ncu split rc=$?"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:paged_gqa_decode_cluster --launch-skip 4 -c 1 -o gpurun_out/c6_cluster_tp8_b1_16k -f python tools/k1_split_trace.py --variant cluster --batch 1 --hq 8 --hkv 1 --seq 16384 > gpurun_out/c6_ncu_cluster.log 2>&1; echo "ncu cluster rc=$?"
tail -3 gpurun_out/c6_ncu_split.log gpurun_out/c6_ncu_cluster.log
ls -la gpurun_out/
