# block order inside a brick: z-fastest (shipped) vs boustrophedon (consecutive blocks share a face), 64M and 8M
for v in "" _snake; do
  SPHG_LIB=libsphg$v.so timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abs$v.log 2>&1
  tail -1 gpurun_out/abs$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5 lib$v', round(d['ms_per_step'],2), 'rebuild', round(d['rebuild_ms'],1), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid','extrapolate','forces_rigid')})"
done
SPHG_LIB=libsphg_snake.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "nlist or full_size or sm_local" -p no:cacheprovider > gpurun_out/abs_pytest.log 2>&1; tail -2 gpurun_out/abs_pytest.log
echo done
