timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "nlist or cells or full_size_parity" > gpurun_out/vb_t.log 2>&1; tail -3 gpurun_out/vb_t.log
timeout 900 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/vb_b.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/vb_b.log').read().splitlines()[-1]); print('ms/step', d['ms_per_step'], 'rebuild_ms', d['rebuild_ms'], 'stage', d['stage_ms']['rebuild'])"
