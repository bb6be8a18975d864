timeout 600 python -m pytest tests -m gpu -q -rf -x 2>&1 | tail -5 > gpurun_out/pytest5.log
for LIB in libsphg.so libsphg_tight.so; do for G in 4 8; do
  SPHG_LIB=$LIB SPHG_GROUP_DENSITY=$G SPHG_GROUP_FORCES=$G timeout 300 python bench.py --nside 200 --spheres 2500 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/sweepc_${LIB}_G$G.log 2>&1
done; done
echo done
