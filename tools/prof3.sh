CMD="python bench.py --nside 128 --spheres 655 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_forces_fluid" -s 1 -c 1 -o gpurun_out/prof_r01f $CMD > gpurun_out/ncu_f.log 2>&1
echo done
