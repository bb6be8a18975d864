CMD="python bench.py --nside 128 --spheres 655 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_forces_fluid|k_density" -s 2 -c 2 -o gpurun_out/prof_r01d $CMD > gpurun_out/ncu_d.log 2>&1
echo done
