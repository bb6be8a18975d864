timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_golden.py tests/test_output.py tests/test_gpu_decomposition.py -q -p no:cacheprovider -k "transition or melt or dissolve or c2 or c4 or golden or roundtrip or speculation or graph or event or full_size" > gpurun_out/vm_t.log 2>&1; tail -3 gpurun_out/vm_t.log
for r in 1 2; do
timeout 900 python tools/bench_melt.py 40 > gpurun_out/melt_a$r.log 2>&1; grep -o '"case": "[a-z0-9_]*", "n": [0-9]*, "ms_per_step": [0-9.]*' gpurun_out/melt_a$r.log
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/melt_l_a.csv python tools/melt_steps.py > gpurun_out/melt_ncu_a.log 2>&1
