timeout 900 python tools/bench_melt.py 20 > gpurun_out/melt2.log 2>&1; tail -2 gpurun_out/melt2.log
SPHG_REPART_ALL=1 timeout 900 python tools/bench_melt.py 20 > gpurun_out/melt3.log 2>&1; tail -2 gpurun_out/melt3.log
