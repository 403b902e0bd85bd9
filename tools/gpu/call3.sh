mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q -p no:cacheprovider -k "cluster" > gpurun_out/c3_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/c3_pytest.log
timeout 900 python tools/k1_variant_sweep.py > gpurun_out/c3_variants.md 2> gpurun_out/c3_variants.err; echo "sweep rc=$?"
cat gpurun_out/c3_variants.md; tail -5 gpurun_out/c3_variants.err
