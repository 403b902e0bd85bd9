# Decoder step (70B TP8 shard, B=32, 64K) vs K1 split length (OFB_K1_BPS): one-wave 2/SM plans vs the cost model's 256
mkdir -p gpurun_out/decbps
for bps in default 128 342 456 512; do
  if [ $bps = default ]; then E=""; else E="OFB_K1_BPS=$bps"; fi
  env $E timeout 600 python tools/decoder_probe.py --tp 8 --prompt 65528 --steps 6 --c1 k6 > gpurun_out/decbps/bps_$bps.jsonl 2>&1; echo "bps=$bps rc=$? $(tail -1 gpurun_out/decbps/bps_$bps.jsonl | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(sorted(d["step_ms"][1:])[2])')"
done
