timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/h_pytest.log 2>&1; tail -5 gpurun_out/h_pytest.log
