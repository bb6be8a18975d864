run() { env "$@" timeout 300 python bench.py --nside 200 --spheres 2500 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline; }
run SPHG_PERSIST_BLOCKS=0 > gpurun_out/p_base.log 2>&1
run SPHG_PERSIST_BLOCKS=740 > gpurun_out/p_740.log 2>&1
run SPHG_PERSIST_BLOCKS=1480 > gpurun_out/p_1480.log 2>&1
run SPHG_PERSIST_BLOCKS=148 SPHG_PERSIST_THREADS=640 > gpurun_out/p_148x640.log 2>&1
run SPHG_PERSIST_BLOCKS=296 SPHG_PERSIST_THREADS=640 > gpurun_out/p_296x640.log 2>&1
echo done
