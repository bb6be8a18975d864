# ncu full-set capture of k_density at 64M (the r02 pair-kernel capture window missed it)
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_density" -c 1 -o gpurun_out/prof_${1:-r02}_density $CMD > gpurun_out/ncu_d64.log 2>&1
echo done
