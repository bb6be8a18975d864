run() { env "$@" timeout 600 python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline; }
run SPHG_ROW_HINT=0 > gpurun_out/h0.log 2>&1
run SPHG_ROW_HINT=1 > gpurun_out/h1.log 2>&1
echo done
