CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 1800 ncu --set full --clock-control none --import-source on \
  -k regex:"k_forces_fluid|k_density|k_forces_rigid|k_extrapolate" -s 8 -c 9 \
  -o gpurun_out/prof_r01f $CMD > gpurun_out/ncu_f_r01f.log 2>&1
echo done
