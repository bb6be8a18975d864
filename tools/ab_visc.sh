# fluid forces with the viscous sum split (u_i out of the loop's registers) at 7 resident blocks per SM (72 registers,
# 12 B spilled) against the shipped kernel (80 registers, 6 blocks), 64M
for v in "" _vs7; do
  SPHG_LIB=libsphg$v.so timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abv$v.log 2>&1
  tail -1 gpurun_out/abv$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('lib$v', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid','extrapolate','forces_rigid')})"
done
echo done
