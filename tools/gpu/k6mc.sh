# K6 batch-split pairs with W multicast (mc) vs split-K pairs: parity, timing, sanitizers
timeout 900 python -m pytest tests/test_oproj_gpu.py tests/test_decoder_gpu.py -x -q -p no:cacheprovider > gpurun_out/k6mc_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/k6mc_pytest.log
fmt='import sys,json
for l in sys.stdin:
  try: d=json.loads(l); print(d["shape"], round(d["k6_us"],2), round(d["cublas_us"],2), round(d["speedup_vs_cublas"],3))
  except Exception: print(l.strip()[:200])'
for mc in 1 0; do echo "== mc $mc"; OFB_K6_MC=$mc timeout 300 python tools/oproj_bench.py --no-emulated 2>&1 | python -c "$fmt"; done
for mc in 1 0; do echo "== decoder mc $mc"; OFB_K6_MC=$mc timeout 300 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 5 2>&1 | tail -1 | cut -c80-200; done
for t in synccheck racecheck memcheck; do r=$(timeout 300 compute-sanitizer --tool $t python tools/k6_sync_case.py 32 1024 8192 2>&1 | grep -E "SUMMARY" | head -1); echo "$t: $r"; done
