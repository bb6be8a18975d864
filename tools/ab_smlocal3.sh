# SM-local pair kernels: lanes per particle and L1 carveout (64M, 30 steps)
run() {  # name env...
  name=$1; shift
  env SPHG_LIB=libsphg_g.so "$@" timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab3_$name.log 2>&1
  tail -1 gpurun_out/ab3_$name.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$name', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid','extrapolate','forces_rigid')})"
}
run base SPHG_X=0
run f8 SPHG_GROUP_FORCES=8
run d8 SPHG_GROUP_DENSITY=8
run carve0 SPHG_SMEM_CARVEOUT=0
echo done
