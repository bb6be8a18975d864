timeout 600 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -5 > gpurun_out/pytest6.log
for U in 1 2; do for G in 2 4 8; do
  SPHG_UNROLL_FORCES=$U SPHG_GROUP_DENSITY=$G SPHG_GROUP_FORCES=$G timeout 300 python bench.py --nside 200 --spheres 2500 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/sweepd_U${U}_G$G.log 2>&1
done; done
echo done
