run() { env "$@" timeout 900 python bench.py --steps 100 --warmup 3 --no-e2e --no-cpu-baseline; }
for v in default exactq; do
  if [ $v = default ]; then run > gpurun_out/eq_$v.log 2>&1; else run SPHG_LIB=libsphg_$v.so > gpurun_out/eq_$v.log 2>&1; fi
  python -c "import json; d=json.loads(open('gpurun_out/eq_$v.log').read().strip().splitlines()[-1]); s=d['stage_ms']; print('$v', round(d['ms_per_step'],2), {k: round(v,3) for k,v in s.items() if v})"
done
