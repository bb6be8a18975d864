timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/j_bench.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/j_bench.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['stage_ms'])"
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/j_pytest.log 2>&1; tail -3 gpurun_out/j_pytest.log
