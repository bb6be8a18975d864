# Profile capture for one round: plain run (must exit 0), launch list of the same command,
# then one full-set capture of the top kernels.  usage: bash tools/prof_round.sh TAG
TAG=${1:-r01b}
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_l_$TAG.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_forces_fluid|k_density|k_build_nlist_cells|k_forces_rigid" -s 6 -c 4 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_f_$TAG.log 2>&1
echo done
