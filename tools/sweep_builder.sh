# Verlet-builder variants (tools/build_variants.py): rebuild_ms of the bench line at 64M
for v in ${VARIANTS:-default orig p16 p20}; do
  if [ $v = default ]; then L=libsphg.so; else L=libsphg_$v.so; fi
  SPHG_LIB=$L timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sb_$v.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/sb_$v.log').read().splitlines()[-1]); print('$v', 'rebuild_ms', round(d['rebuild_ms'],2), 'ms/step', round(d['ms_per_step'],2))" 2>/dev/null || tail -2 gpurun_out/sb_$v.log
done
