mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_fullsize_gpu.py -x -q -p no:cacheprovider > gpurun_out/c19_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/c19_pytest.log
timeout 900 python tools/k1_variant_sweep.py > gpurun_out/c19_variants_wide.md 2> gpurun_out/c19_variants_wide.err; echo "sweep rc=$?"
OFB_K1_WIDE=0 timeout 900 python tools/k1_variant_sweep.py --quick > gpurun_out/c19_variants_narrow.md 2> gpurun_out/c19_variants_narrow.err; echo "sweep2 rc=$?"
for shape in "1 8 1 16384" "1 32 8 4096"; do
  set -- $shape
  echo "== split B=$1 hq=$2 hkv=$3 seq=$4"
  timeout 120 python tools/k1_split_trace.py --variant split --batch $1 --hq $2 --hkv $3 --seq $4
done > gpurun_out/c19_trace.txt 2>&1
timeout 600 python tools/k1_sweep.py > gpurun_out/c19_k1_sweep.md 2> gpurun_out/c19_k1_sweep.err; echo "k1 sweep rc=$?"
timeout 1500 python bench.py --config cfg3 --cfg3-rate 300 --cfg3-budget-blocks 262144 > gpurun_out/c19_cfg3_sat.json 2> gpurun_out/c19_cfg3_sat.err; echo "cfg3 sat rc=$?"
tail -c 1200 gpurun_out/c19_cfg3_sat.err
