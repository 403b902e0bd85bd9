# cfg2r (8B, B=16, 32K, every layer resident): K1 late consumer wait on (default) vs off (OFB_K1_LATE=0), same box, twice
mkdir -p gpurun_out/cfg2r
for i in 1 2; do
  OFB_K1_LATE=0 timeout 600 python bench.py --config cfg2r --no-cpu-baseline > gpurun_out/cfg2r/late0_$i.json 2> gpurun_out/cfg2r/late0_$i.err
  timeout 600 python bench.py --config cfg2r --no-cpu-baseline > gpurun_out/cfg2r/late1_$i.json 2> gpurun_out/cfg2r/late1_$i.err
done
echo done
