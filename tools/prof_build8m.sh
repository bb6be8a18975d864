# ncu full-set + source capture of the Verlet builder on one GPU's weak-scaling share (C5 200^3 = 8M)
CMD="python bench.py --nside 200 --spheres 2500 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/pb_plain.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_build_nlist_cells" -c 1 -o gpurun_out/prof_${1:-r02}_build8m $CMD > gpurun_out/ncu_b8.log 2>&1
echo done
