# speculative force chain (default) vs the flag readback before it (SPHG_SPECULATE=0)
for cfg in c1 c2 c3 c5; do for v in 1 0; do
  st=300; [ $cfg = c5 ] && st=50
  SPHG_SPECULATE=$v timeout 900 python bench.py --config $cfg --steps $st --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/spec_${cfg}_$v.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/spec_${cfg}_$v.log').read().strip().splitlines()[-1]); print('$cfg speculate=$v', round(d['ms_per_step'],4), d['rebuilds_in_timed_region'])"
done; done
