# Decoder step at 64K: balanced split lengths (242 = ceil(4097/17)) vs 256 / 512, and a prompt whose steps stay inside 4096 blocks
mkdir -p gpurun_out/decbps3
run() { # batch prompt bps
  if [ $3 = default ]; then E=""; else E="OFB_K1_BPS=$3"; fi
  env $E timeout 600 python tools/decoder_probe.py --tp 8 --batch $1 --prompt $2 --steps 6 --c1 k6 > gpurun_out/decbps3/b$1_p$2_bps$3.jsonl 2>&1
  echo "B=$1 prompt=$2 bps=$3 $(tail -1 gpurun_out/decbps3/b$1_p$2_bps$3.jsonl | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(sorted(d["step_ms"][1:])[2])')"
}
run 32 65528 default; run 32 65528 242; run 32 65528 512; run 32 65528 410
run 32 65400 default; run 32 65400 512
