timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/i_pytest.log 2>&1; tail -3 gpurun_out/i_pytest.log
bash tools/bench_secondary.sh
