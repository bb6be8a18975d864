timeout 1200 python -m pytest tests/test_gpu_decomposition.py -q -p no:cacheprovider > gpurun_out/v2_dec.log 2>&1; tail -5 gpurun_out/v2_dec.log
