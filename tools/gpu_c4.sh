set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "c4 or powder or golden or graph_replay" > gpurun_out/c4_pytest.log 2>&1; tail -5 gpurun_out/c4_pytest.log
timeout 900 python bench.py --config c4 --steps 200 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c4_bench.log 2>&1; tail -1 gpurun_out/c4_bench.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/c4_allgpu.log 2>&1; tail -3 gpurun_out/c4_allgpu.log
