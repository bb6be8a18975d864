# secondary bench lines (BASELINE sizes) + the headline; one JSON line each into gpurun_out/sec_*.log
for cfg in c1 c2 c3 dissolve paper46 c4; do
  timeout 900 python bench.py --config $cfg --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/sec_$cfg.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sec_$cfg.log').read().strip().splitlines()[-1]); print('$cfg', d['config']['particles'], round(d['ms_per_step'],4), '%.3e' % d['value'])"
done
