timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/sp2_pytest.log 2>&1; tail -3 gpurun_out/sp2_pytest.log
for cfg in c2 dissolve c4; do for v in 1 0; do
  st=300; [ $cfg = c4 ] && st=100
  SPHG_SPECULATE=$v timeout 900 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sp2_${cfg}_$v.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/sp2_${cfg}_$v.log').read().strip().splitlines()[-1]); print('$cfg speculate=$v', round(d['ms_per_step'],4))"
done; done
