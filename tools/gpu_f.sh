timeout 900 python -m pytest tests -x -q -m gpu -k "step_download or cpp_dropin" > gpurun_out/f_pytest.log 2>&1; tail -3 gpurun_out/f_pytest.log
timeout 1200 python bench.py > gpurun_out/f_bench.log 2>&1; tail -1 gpurun_out/f_bench.log
