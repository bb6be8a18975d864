# steal-scan variants at the weak-scaling share (C5 200^3 = 8M) and paper46 (3.8M)
run() {  # name lib env
  SPHG_LIB=$2 env $3 timeout 900 python bench.py --nside 200 --spheres 2500 --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab6_$1.log 2>&1
  tail -1 gpurun_out/ab6_$1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5_200 $1', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid','extrapolate','forces_rigid')})"
  SPHG_LIB=$2 env $3 timeout 900 python bench.py --config paper46 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab6_p46_$1.log 2>&1
  tail -1 gpurun_out/ab6_p46_$1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('paper46 $1', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid','extrapolate','forces_rigid')})"
}
run flat libsphg_seq.so SPHG_SM_LOCAL=0
run seq libsphg_seq.so SPHG_X=0
run new libsphg.so SPHG_X=0
run lb libsphg_lb.so SPHG_X=0
echo done
