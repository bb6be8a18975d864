timeout 1500 python -m pytest tests -q -m gpu -k full_size > gpurun_out/m_pytest.log 2>&1; tail -4 gpurun_out/m_pytest.log
bash tools/prof_round.sh r01f
bash tools/prof_build64.sh r01f
