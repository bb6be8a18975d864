# Profile capture for one round: plain run (must exit 0), launch list of the same command,
# then one full-set capture of each top kernel.  usage: bash tools/prof_round.sh TAG
TAG=${1:-r01}
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_l_$TAG.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on \
  -k regex:"k_forces_fluid|k_density|k_forces_rigid|k_build_nlist_cells|k_extrapolate" -s 8 -c 9 \
  -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_f_$TAG.log 2>&1
echo done
