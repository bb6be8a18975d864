# steal scan variants: lane-parallel (default), sequential atomics (seq), default + 12 blocks/SM density (lb)
for v in "" _seq _lb; do
  SPHG_LIB=libsphg$v.so timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab5_c5$v.log 2>&1
  tail -1 gpurun_out/ab5_c5$v.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c5$v', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid','extrapolate','forces_rigid')})"
  for cfg in c3 c4; do
    SPHG_LIB=libsphg$v.so timeout 900 python bench.py --config $cfg --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ab5_$cfg$v.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab5_$cfg$v.log').read().strip().splitlines()[-1]); print('$cfg$v', d['config']['particles'], round(d['ms_per_step'],4), '%.3e' % d['value'])"
  done
done
echo done
