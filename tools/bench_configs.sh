# secondary measurements on the other BASELINE configs at their BASELINE sizes
for cfg in c2 c3 c1 dissolve; do
  timeout 900 python bench.py --config $cfg --steps 50 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bcfg_$cfg.log 2>&1
done
echo done
