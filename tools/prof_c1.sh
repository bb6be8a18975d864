# launch list of the C1 bench (32^3): where a 0.15 ms step goes
CMD="python bench.py --config c1 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/c1_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $CMD > gpurun_out/ncu_c1.log 2>&1
tail -1 gpurun_out/c1_plain.log | cut -c1-300
