# SM-local pair kernels: in-brick cell order and L1 eviction hints (64M, 30 steps)
run() {  # name lib
  SPHG_LIB=$2 SPHG_SM_LOCAL=3 timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab2_$1.log 2>&1
  tail -1 gpurun_out/ab2_$1.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$1', round(d['ms_per_step'],2), 'rebuild', round(d.get('rebuild_ms',0),1), {k: round(v,2) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid','extrapolate','forces_rigid')})"
}
run base libsphg.so
run sub libsphg_sub.so
run rowef libsphg_rowef.so
run recel libsphg_recel.so
run sub_rowef libsphg_sub_rowef.so
echo done
