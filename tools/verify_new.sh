timeout 900 python -m pytest tests/test_gpu_decomposition.py -q -p no:cacheprovider -k "bench_two_ranks" > gpurun_out/v3.log 2>&1; tail -3 gpurun_out/v3.log
timeout 600 python bench.py --nside 64 --spheres 20 --steps 3 --warmup 3 --cpu-nside 24 > gpurun_out/v3b.log 2>&1; tail -c 600 gpurun_out/v3b.log
