run() { env "$@" timeout 300 python bench.py --nside 200 --spheres 2500 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline; }
run SPHG_UNROLL_FORCES=1 > gpurun_out/s_u1.log 2>&1
run SPHG_UNROLL_FORCES=4 > gpurun_out/s_u4.log 2>&1
run SPHG_UNROLL_FORCES=4 SPHG_GROUP_FORCES=8 > gpurun_out/s_u4g8.log 2>&1
run SPHG_UNROLL_FORCES=1 SPHG_GROUP_FORCES=8 > gpurun_out/s_u1g8.log 2>&1
echo done
