# store-size sweep of the C5 workload (sphere density of C5): 200^3 = 8M (the weak-scaling share of one
# GPU at N = 8), 400^3 = 64M (the headline), 440^3 = 85M (about the largest store that fits one B200)
for ns in 200 440; do
  sp=$(python -c "print(int(round(20000 * ($ns / 400.0) ** 3)))")
  timeout 1200 python bench.py --nside $ns --spheres $sp --steps 50 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/size_$ns.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/size_$ns.log').read().strip().splitlines()[-1]); print($ns, d['config']['particles'], round(d['ms_per_step'],3), '%.4e' % d['value'], d['device_memory_gb'], d['rebuilds_in_timed_region'])"
done
