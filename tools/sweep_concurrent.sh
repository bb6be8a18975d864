# rigid force pass on a second stream (default) vs serialised
run() { env "$@" timeout 900 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu-baseline; }
for v in 1 0; do
  run SPHG_CONCURRENT_RIGID=$v > gpurun_out/conc_$v.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/conc_$v.log').read().strip().splitlines()[-1]); print('concurrent=$v', round(d['ms_per_step'],3), '%.4e' % d['value'])"
done
