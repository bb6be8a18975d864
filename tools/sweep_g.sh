# group width sweep for the pair kernels (64M, steady state)
run() { env "$@" timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline; }
run SPHG_GROUP_DENSITY=8 SPHG_GROUP_FORCES=8 > gpurun_out/g88.log 2>&1
run SPHG_GROUP_DENSITY=2 SPHG_GROUP_FORCES=2 > gpurun_out/g22.log 2>&1
run SPHG_GROUP_DENSITY=4 SPHG_GROUP_FORCES=4 > gpurun_out/g44.log 2>&1
echo done
