timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/d_pytest.log 2>&1; tail -3 gpurun_out/d_pytest.log
for v in 1; do
  timeout 600 python bench.py --config dissolve --steps 300 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/d_dissolve.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/d_dissolve.log').read().strip().splitlines()[-1]); print('dissolve', round(d['ms_per_step'],4))"
done
