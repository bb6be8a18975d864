timeout 900 python -m pytest tests -x -q -m gpu -k "c4 or powder or heat_flux or graph_replay" > gpurun_out/c4b_pytest.log 2>&1; tail -5 gpurun_out/c4b_pytest.log
