#!/bin/bash
# K6 residual prefetch: parity, sanitizer on the fused-residual case, decoder probe and cfg4-serve TP8
timeout 900 python -m pytest tests/test_oproj_gpu.py tests/test_decoder_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for t in synccheck racecheck memcheck; do r=$(timeout 600 compute-sanitizer --tool $t python tools/sanitize_case.py 2>&1 | grep -E "SUMMARY" | head -1); echo "$t: $r"; done
mkdir -p gpurun_out/res
for i in 1 2; do timeout 600 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 6 --c1 k6 2>&1 | grep step_ms; done
timeout 1500 python bench.py --config cfg4-serve --tp-emulate 8 > gpurun_out/res/cfg4_serve_tp8.json 2> gpurun_out/res/cfg4_serve_tp8.err; echo "cfg4 rc=$?"
