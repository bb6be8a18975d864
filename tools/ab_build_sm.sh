# Verlet builder on an SM-local persistent grid (bit 5) at 64M: rebuild_ms; list parity with it forced on small cases
for m in 31 63; do
  SPHG_SM_LOCAL=$m timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/abb_$m.log 2>&1
  tail -1 gpurun_out/abb_$m.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('sm_local=$m', round(d['ms_per_step'],2), 'rebuild_ms', round(d['rebuild_ms'],2))"
done
SPHG_SM_LOCAL=63 SPHG_SM_LOCAL_MIN=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "nlist or sm_local or full_size" -p no:cacheprovider > gpurun_out/abb_pytest.log 2>&1; tail -3 gpurun_out/abb_pytest.log
echo done
