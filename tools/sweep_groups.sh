timeout 900 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > gpurun_out/pytest4.log
for G in 8 16 32; do
  SPHG_GROUP_DENSITY=$G SPHG_GROUP_FORCES=$G timeout 300 python bench.py --nside 200 --spheres 2500 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/sweep_G$G.log 2>&1
done
echo done
