CMD="python bench.py --nside 200 --spheres 2500 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plainb.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_build_nlist_cells" -c 1 -o gpurun_out/prof_build3 $CMD > gpurun_out/ncu_b3.log 2>&1
echo done
