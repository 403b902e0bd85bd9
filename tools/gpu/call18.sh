mkdir -p gpurun_out
timeout 2400 python bench.py --config cfg3 > gpurun_out/c18_cfg3_40g.json 2> gpurun_out/c18_cfg3_40g.err; echo "cfg3 40g rc=$?"
tail -c 1500 gpurun_out/c18_cfg3_40g.err
timeout 600 python -m pytest tests/test_decoder_gpu.py tests/test_oproj_gpu.py -x -q -p no:cacheprovider > gpurun_out/c18_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/c18_pytest.log
timeout 600 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 4 > gpurun_out/c18_probe_tp8.json 2>&1; tail -2 gpurun_out/c18_probe_tp8.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/c18_probe_tp8_launches.csv python tools/decoder_probe.py --tp 8 --prompt 4088 --steps 3 --profile-last > /dev/null 2>&1; echo "ncu rc=$?"
