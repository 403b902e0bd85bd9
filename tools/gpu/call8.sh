mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q -p no:cacheprovider -k "not torch" > gpurun_out/c10_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/c10_pytest.log
for v in split cluster; do
for shape in "1 8 1 16384" "1 32 8 4096" "4 8 1 16384" "1 8 1 65536"; do
  set -- $shape
  echo "== $v B=$1 hq=$2 hkv=$3 seq=$4"
  timeout 120 python tools/k1_split_trace.py --variant $v --batch $1 --hq $2 --hkv $3 --seq $4
done; done > gpurun_out/c10_trace.txt 2>&1
timeout 900 python tools/k1_variant_sweep.py > gpurun_out/c10_variants.md 2> gpurun_out/c10_variants.err; echo "sweep rc=$?"
cat gpurun_out/c10_variants.md
