# end-of-round evidence: parity suite, smoke, the default bench line (with e2e and the CPU leg),
# the reference arm, and the secondary configs
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/fin_pytest.log 2>&1; tail -2 gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
timeout 1200 python bench.py > gpurun_out/fin_bench.log 2>&1; tail -1 gpurun_out/fin_bench.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.log 2>&1; tail -1 gpurun_out/fin_ref.log | cut -c1-300
bash tools/bench_secondary.sh
