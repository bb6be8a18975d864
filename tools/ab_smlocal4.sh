# SM-local grids: size threshold and the cheaper steal scan (secondary configs), extrapolation / rigid at 64M
sec() {  # name cfg env...
  name=$1; cfg=$2; shift; shift
  env "$@" timeout 900 python bench.py --config $cfg --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab4_$name.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab4_$name.log').read().strip().splitlines()[-1]); print('$name', d['config']['particles'], round(d['ms_per_step'],4), '%.3e' % d['value'])"
}
sec c1_default c1 SPHG_X=0
sec c1_flat c1 SPHG_SM_LOCAL=0
sec c1_forced c1 SPHG_SM_LOCAL_MIN=0
sec c2_default c2 SPHG_X=0
sec c2_forced c2 SPHG_SM_LOCAL_MIN=0
sec c3_default c3 SPHG_X=0
sec c3_flat c3 SPHG_SM_LOCAL=0
sec c3_all c3 SPHG_SM_LOCAL=15
sec p46_default paper46 SPHG_X=0
sec p46_flat paper46 SPHG_SM_LOCAL=0
sec p46_all paper46 SPHG_SM_LOCAL=15
sec c4_default c4 SPHG_X=0
sec c4_flat c4 SPHG_SM_LOCAL=0
sec c4_all c4 SPHG_SM_LOCAL=15
for m in 3 15; do
  SPHG_SM_LOCAL=$m timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab4_c5_$m.log 2>&1
  tail -1 gpurun_out/ab4_c5_$m.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5 sm_local=$m', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid','extrapolate','forces_rigid')})"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "sm_local or graph or speculation" -p no:cacheprovider > gpurun_out/ab4_pytest.log 2>&1; tail -3 gpurun_out/ab4_pytest.log
echo done
