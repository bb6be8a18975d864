run() { env "$@" timeout 300 python bench.py --nside 200 --spheres 2500 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline; }
run SPHG_LIB=libsphg.so > gpurun_out/r_base.log 2>&1
run SPHG_LIB=libsphg_mb6.so > gpurun_out/r_mb6.log 2>&1
run SPHG_LIB=libsphg_mb7.so > gpurun_out/r_mb7.log 2>&1
run SPHG_GROUP_FORCES=2 > gpurun_out/r_g2.log 2>&1
run SPHG_LIB=libsphg_mb6.so SPHG_GROUP_FORCES=2 > gpurun_out/r_mb6g2.log 2>&1
echo done
