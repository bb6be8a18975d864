timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3 > gpurun_out/chk_pytest.log
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain64b.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_build|k_reorder|k_down|k_up|k_scan|k_keys|k_cell|k_kind|k_rigid|k_body_ranges|k_idx" --log-file gpurun_out/launches_rebuild.csv $CMD > gpurun_out/ncu_rb.log 2>&1
echo done
