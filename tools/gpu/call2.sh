mkdir -p gpurun_out
set -x
timeout 900 python -m pytest tests/test_torch_ops.py tests/test_kernels_gpu.py -x -q -p no:cacheprovider > gpurun_out/c2_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/c2_pytest.log
timeout 900 python bench.py --config cfg4-serve --tp-emulate 4 > gpurun_out/c2_cfg4_tp4.json 2> gpurun_out/c2_cfg4_tp4.err; echo "cfg4 tp4 rc=$?"
tail -c 1500 gpurun_out/c2_cfg4_tp4.json; tail -5 gpurun_out/c2_cfg4_tp4.err | cut -c1-300
timeout 600 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 4 > gpurun_out/c2_probe_tp8.json 2>&1; echo "probe rc=$?"
tail -5 gpurun_out/c2_probe_tp8.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/c2_probe_tp8_launches.csv python tools/decoder_probe.py --tp 8 --prompt 4088 --steps 2 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/c2_ref.json 2> gpurun_out/c2_ref.err; echo "ref rc=$?"
tail -c 1500 gpurun_out/c2_ref.json
