set -x
timeout 600 python -m pytest tests -x -q -m gpu -k graph_replay > gpurun_out/t_graph.log 2>&1
tail -3 gpurun_out/t_graph.log
for cfg in c1 c2 c3 dissolve; do
  for g in 1 0; do
    SPHG_GRAPHS=$g timeout 600 python bench.py --config $cfg --steps 200 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bg_${cfg}_$g.log 2>&1
    tail -1 gpurun_out/bg_${cfg}_$g.log | cut -c1-200
  done
done
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
