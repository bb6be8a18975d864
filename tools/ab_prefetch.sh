# next-round record prefetch into L1 in the fluid forces row walk (64M)
for v in "" _pf; do
  SPHG_LIB=libsphg$v.so timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abpf$v.log 2>&1
  tail -1 gpurun_out/abpf$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('lib$v', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid','extrapolate','forces_rigid')})"
done
echo done
