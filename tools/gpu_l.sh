bash tools/sweep_old.sh
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/l_pytest.log 2>&1; tail -3 gpurun_out/l_pytest.log
