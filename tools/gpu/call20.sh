mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_oproj_gpu.py -x -q -p no:cacheprovider > gpurun_out/c20_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/c20_pytest.log
timeout 600 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 4 > gpurun_out/c20_probe_tp8.json 2>&1; tail -2 gpurun_out/c20_probe_tp8.json
timeout 600 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 4 --c1 nccl > gpurun_out/c20_probe_tp8_nccl.json 2>&1; tail -2 gpurun_out/c20_probe_tp8_nccl.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/c20_probe_tp8_launches.csv python tools/decoder_probe.py --tp 8 --prompt 4088 --steps 3 --profile-last > /dev/null 2>&1; echo "ncu rc=$?"
for tp in 8 4 2 1; do
  timeout 1200 python bench.py --config cfg4-serve --tp-emulate $tp > gpurun_out/c20_cfg4_tp$tp.json 2> gpurun_out/c20_cfg4_tp$tp.err; echo "cfg4 tp$tp rc=$?"; tail -c 400 gpurun_out/c20_cfg4_tp$tp.json
done
