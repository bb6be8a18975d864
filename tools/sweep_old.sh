run() { env "$@" timeout 900 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu-baseline; }
for v in default old; do
  if [ $v = default ]; then run > gpurun_out/old_$v.log 2>&1; else run SPHG_LIB=libsphg_$v.so > gpurun_out/old_$v.log 2>&1; fi
  python -c "import json; d=json.loads(open('gpurun_out/old_$v.log').read().strip().splitlines()[-1]); s=d['stage_ms']; print('$v', round(d['ms_per_step'],2), 'extrap', round(s['extrapolate'],3), 'rigid', round(s['forces_rigid'],3), 'fluid', round(s['forces_fluid'],2), 'dens', round(s['density'],2))"
done
