# Verlet-build variants (tools/build_variants.py) at 8M and 64M: rebuild_ms per variant
for v in w1s512 w2s256 w4s256 w2s384 w4s128 w2s256r80; do
  SPHG_LIB=libsphg_$v.so timeout 300 python bench.py --nside 200 --spheres 2500 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sb8_$v.log 2>&1
done
for v in w1s512 w2s384 w2s256r80; do
  SPHG_LIB=libsphg_$v.so timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sb64_$v.log 2>&1
done
echo done
