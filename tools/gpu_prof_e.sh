timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/e_pytest.log 2>&1; tail -3 gpurun_out/e_pytest.log
bash tools/prof_round.sh r01e
bash tools/prof_build64.sh r01e
ls -la gpurun_out/
