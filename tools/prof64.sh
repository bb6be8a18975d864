CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain64.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01_64m.csv $CMD > gpurun_out/ncu_l64.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_forces_fluid|k_density" -s 8 -c 2 -o gpurun_out/prof_r01_64m $CMD > gpurun_out/ncu_f64.log 2>&1
echo done
