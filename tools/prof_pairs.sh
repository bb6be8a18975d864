# G sweep (4/8) + ncu full capture of density/forces at 128^3 (G=8)
for G in 4 8; do
  SPHG_GROUP_DENSITY=$G SPHG_GROUP_FORCES=$G timeout 300 python bench.py --nside 200 --spheres 2500 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/sweepb_G$G.log 2>&1
done
CMD="python bench.py --nside 128 --spheres 655 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_forces_fluid|k_density|k_extrapolate|k_forces_rigid" -s 4 -c 4 -o gpurun_out/prof_r01c $CMD > gpurun_out/ncu_c.log 2>&1
echo done
