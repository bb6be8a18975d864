# A/B of the SM-local persistent pair kernels at 64M (SPHG_SM_LOCAL: 1 forces, 2 density, 3 both)
for m in 0 1 3; do
  SPHG_SM_LOCAL=$m timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_sm_$m.log 2>&1
  tail -1 gpurun_out/ab_sm_$m.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('sm_local=$m', d['ms_per_step'], {k: round(v,2) for k,v in d['stage_ms'].items()})"
done
SPHG_SM_LOCAL=3 timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/ab_sm_pytest.log 2>&1; tail -3 gpurun_out/ab_sm_pytest.log
echo done
