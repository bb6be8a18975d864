run() { env "$@" timeout 300 python bench.py --nside 200 --spheres 2500 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline; }
run SPHG_UNROLL_FORCES=1 > gpurun_out/q_u1.log 2>&1
run SPHG_UNROLL_FORCES=3 > gpurun_out/q_u3.log 2>&1
run SPHG_UNROLL_FORCES=1 SPHG_GROUP_FORCES=8 SPHG_GROUP_DENSITY=8 > gpurun_out/q_u1g8.log 2>&1
run SPHG_UNROLL_FORCES=3 SPHG_GROUP_FORCES=8 > gpurun_out/q_u3g8.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2 > gpurun_out/q_pytest.log
echo done
