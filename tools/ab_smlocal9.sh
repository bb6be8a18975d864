# resident blocks per SM of the persistent grids (fewer particles in flight per L1) at 64M
for b in 12 5 4 8; do
  SPHG_SM_BLOCKS=$b timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab9_$b.log 2>&1
  tail -1 gpurun_out/ab9_$b.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('blocks<=$b', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid','extrapolate','forces_rigid')})"
done
echo done
