# density pass: two gathers in flight at 12 blocks/SM (shipped) vs one gather at 16 blocks/SM (32 registers), 64M and 8M
for v in "" _d16 _d12s; do
  SPHG_LIB=libsphg$v.so timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abd$v.log 2>&1
  tail -1 gpurun_out/abd$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5 lib$v', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid')})"
  SPHG_LIB=libsphg$v.so timeout 900 python bench.py --nside 200 --spheres 2500 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/abd8$v.log 2>&1
  tail -1 gpurun_out/abd8$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5_200 lib$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid')})"
done
echo done
