# Full round check on one B200: parity suite, smoke, default bench line, graph on/off for the small configs.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/v_gpu.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/v_pytest.log 2>&1; tail -3 gpurun_out/v_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; tail -2 gpurun_out/v_smoke.log
timeout 1200 python bench.py > gpurun_out/v_bench.log 2>&1; tail -1 gpurun_out/v_bench.log
for cfg in c1 c2; do
  for g in 1 0; do
    SPHG_GRAPHS=$g timeout 600 python bench.py --config $cfg --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/v_${cfg}_g$g.log 2>&1
    tail -1 gpurun_out/v_${cfg}_g$g.log | cut -c1-200
  done
done
echo done
