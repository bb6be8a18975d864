CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_build_nlist_cells" -c 1 -o gpurun_out/prof_${1:-r01f}_build $CMD > gpurun_out/ncu_b64.log 2>&1
echo done
