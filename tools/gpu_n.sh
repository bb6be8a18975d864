timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/n_pytest.log 2>&1; tail -4 gpurun_out/n_pytest.log
bash tools/sweep_exactq.sh
