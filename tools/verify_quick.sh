# GPU tests, smoke and the default bench line (round check)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v_gpu.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/v_pytest.log 2>&1; tail -4 gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; tail -2 gpurun_out/v_smoke.log
timeout 1800 python bench.py > gpurun_out/v_bench.log 2>&1; tail -1 gpurun_out/v_bench.log | cut -c1-400
echo done
