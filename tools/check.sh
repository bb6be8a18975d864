# parity tests + 8M sweep point + 64M bench (no e2e / cpu baseline) — the standard check after a kernel change
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/chk_pytest.log
timeout 300 python bench.py --nside 200 --spheres 2500 --steps 4 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/chk_8m.log 2>&1
timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/chk_64m.log 2>&1
echo done
