# Steady-state comparison of the current library against a variant build (SPHG_LIB=libsphg_<name>.so,
# e.g. one made by tools/build_variants.py or a library built from an older commit).
# usage: bash tools/compare_lib.sh NAME   (64M, 100 steps, stage-timed breakdown)
V=${1:-old}
run() { env "$@" timeout 900 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu-baseline; }
for v in default $V; do
  if [ $v = default ]; then run > gpurun_out/old_$v.log 2>&1; else run SPHG_LIB=libsphg_$v.so > gpurun_out/old_$v.log 2>&1; fi
  python -c "import json; d=json.loads(open('gpurun_out/old_$v.log').read().strip().splitlines()[-1]); s=d['stage_ms']; print('$v', round(d['ms_per_step'],2), 'extrap', round(s['extrapolate'],3), 'rigid', round(s['forces_rigid'],3), 'fluid', round(s['forces_fluid'],2), 'dens', round(s['density'],2))"
done
