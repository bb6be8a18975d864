# out-of-line steal scan (default lib) against sequential probing (seq lib); forces only (1) or density too (3)
one() {  # label lib mode cfgargs...
  label=$1; lib=$2; mode=$3; shift; shift; shift
  SPHG_LIB=$lib SPHG_SM_LOCAL=$mode timeout 900 python bench.py "$@" --no-e2e --no-cpu-baseline > gpurun_out/ab7_$label.log 2>&1
  tail -1 gpurun_out/ab7_$label.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$label', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stage_ms'].items() if k in ('density','forces_fluid')})"
}
for v in new:libsphg.so seq:libsphg_seq.so; do
  n=${v%%:*}; l=${v##*:}
  for m in 1 3; do
    one c4_${n}_$m $l $m --config c4 --steps 200 --warmup 5
    one c5s_${n}_$m $l $m --nside 200 --spheres 2500 --steps 100 --warmup 5
    one c3_${n}_$m $l $m --config c3 --steps 200 --warmup 5
    one c5_${n}_$m $l $m --steps 30 --warmup 3
  done
done
one c4_flat libsphg.so 0 --config c4 --steps 200 --warmup 5
one c5_flat libsphg.so 0 --steps 30 --warmup 3
echo done
