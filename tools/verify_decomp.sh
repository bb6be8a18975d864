timeout 1200 python -m pytest tests/test_gpu_decomposition.py -q -p no:cacheprovider > gpurun_out/v4_dec.log 2>&1; tail -3 gpurun_out/v4_dec.log
timeout 300 python tools/fp64_peak.py > gpurun_out/fp64.log 2>&1; cp profiles/fp64_peak.json gpurun_out/fp64_peak.json; tail -1 gpurun_out/fp64.log
