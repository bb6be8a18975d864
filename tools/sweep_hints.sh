# L1 eviction-hint variants of the pair kernels (64M steady state, stage-timed breakdown in the JSON)
run() { env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline; }
for v in default rowfirst reclast both; do
  if [ $v = default ]; then run > gpurun_out/hint_$v.log 2>&1; else run SPHG_LIB=libsphg_$v.so > gpurun_out/hint_$v.log 2>&1; fi
  python -c "import json; d=json.loads(open('gpurun_out/hint_$v.log').read().strip().splitlines()[-1]); s=d['stage_ms']; print('$v', round(d['ms_per_step'],2), 'forces_fluid', round(s['forces_fluid'],2), 'density', round(s['density'],2), 'extrap', round(s['extrapolate'],2))"
done
