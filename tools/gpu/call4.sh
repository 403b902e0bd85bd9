mkdir -p gpurun_out
python -c "
from paper_2601_10729_b200 import ops; import torch; torch.cuda.init()
print(ops.cluster_plan(1,1,16384), ops.cluster_plan(1,8,4096))"
timeout 900 python tools/k1_variant_sweep.py > gpurun_out/c4_variants.md 2> gpurun_out/c4_variants.err; echo "sweep rc=$?"
cat gpurun_out/c4_variants.md; tail -3 gpurun_out/c4_variants.err
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q -p no:cacheprovider -k "cluster" > gpurun_out/c4_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/c4_pytest.log
