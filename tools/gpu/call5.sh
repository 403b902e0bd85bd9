mkdir -p gpurun_out
for shape in "1 8 1 16384" "1 8 1 4096" "1 32 8 4096" "4 8 1 16384" "1 32 8 16384"; do
  set -- $shape
  echo "== B=$1 hq=$2 hkv=$3 seq=$4"
  timeout 120 python tools/k1_split_trace.py --batch $1 --hq $2 --hkv $3 --seq $4
done > gpurun_out/c5_split_trace.txt 2>&1
cat gpurun_out/c5_split_trace.txt
