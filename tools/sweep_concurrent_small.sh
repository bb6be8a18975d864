for cfg in c1 c2 c3; do for v in 1 0; do
  SPHG_CONCURRENT_RIGID=$v timeout 600 python bench.py --config $cfg --steps 300 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/concs_${cfg}_$v.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/concs_${cfg}_$v.log').read().strip().splitlines()[-1]); print('$cfg concurrent=$v', round(d['ms_per_step'],4))"
done; done
