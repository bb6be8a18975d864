# block size of the persistent grids (warps per SM at 80 registers: 24 with 128 / 64 threads, 25 with 32), 64M
for t in 128 64 32; do
  SPHG_SM_THREADS=$t timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abt_$t.log 2>&1
  tail -1 gpurun_out/abt_$t.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('threads=$t', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid','extrapolate','forces_rigid')})"
done
echo done
