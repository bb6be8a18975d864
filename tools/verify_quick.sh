set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v_gpu.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/v_pytest.log 2>&1; tail -15 gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; tail -2 gpurun_out/v_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/v_bench.log 2>&1; tail -1 gpurun_out/v_bench.log
echo done
