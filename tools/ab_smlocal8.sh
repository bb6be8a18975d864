# conduction on an SM-local grid (bit 4) at C4, and the bit-identity tests
for m in 15 31; do
  SPHG_SM_LOCAL=$m timeout 900 python bench.py --config c4 --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab8_c4_$m.log 2>&1
  tail -1 gpurun_out/ab8_c4_$m.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c4 sm_local=$m', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items() if v > 0.5})"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_golden.py tests/test_gpu_acceptance.py -q -x -m gpu -p no:cacheprovider > gpurun_out/ab8_pytest.log 2>&1; tail -3 gpurun_out/ab8_pytest.log
echo done
