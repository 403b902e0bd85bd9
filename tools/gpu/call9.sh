mkdir -p gpurun_out
for shape in "1 8 1 16384" "1 8 1 65536"; do
  set -- $shape
  echo "== cluster B=$1 hq=$2 hkv=$3 seq=$4"
  timeout 120 python tools/k1_split_trace.py --variant cluster --batch $1 --hq $2 --hkv $3 --seq $4
done > gpurun_out/c9_trace.txt 2>&1
