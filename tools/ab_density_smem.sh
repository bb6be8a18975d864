# A/B of the TMA cell-staged density (SPHG_DENSITY_SMEM) at 64M + parity tests with it on
SPHG_DENSITY_SMEM=1 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -q -p no:cacheprovider -k "step1 or initialize or stage_by_stage or multistep or golden or full_size or headline" > gpurun_out/ds_t.log 2>&1; tail -2 gpurun_out/ds_t.log
for v in 1 0 1 0; do
  SPHG_DENSITY_SMEM=$v timeout 900 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ds_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ds_$v.log').read().splitlines()[-1]); s=d['stage_ms']; print('smem=$v', 'ms/step', round(d['ms_per_step'],2), 'density', round(s['density'],3))"
done
