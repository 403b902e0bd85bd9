# Decoder step vs K1 split length at 16K / 32K / 64K contexts and B=16 / 32: cost model vs one wave at 2 CTAs/SM
mkdir -p gpurun_out/decbps2
run() { # batch prompt bps
  if [ $3 = default ]; then E=""; else E="OFB_K1_BPS=$3"; fi
  env $E timeout 600 python tools/decoder_probe.py --tp 8 --batch $1 --prompt $2 --steps 6 --c1 k6 > gpurun_out/decbps2/b$1_p$2_bps$3.jsonl 2>&1
  echo "B=$1 prompt=$2 bps=$3 $(tail -1 gpurun_out/decbps2/b$1_p$2_bps$3.jsonl | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(sorted(d["step_ms"][1:])[2])')"
}
run 32 16376 default; run 32 16376 114
run 32 32760 default; run 32 32760 228
run 32 65528 default; run 32 65528 456
run 16 65528 default; run 16 65528 228
run 16 32760 default; run 16 32760 114
