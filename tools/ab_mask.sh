# A/B of the in-range pair masks (density pass -> fluid forces pass) at 64M; the knob SPHG_PAIR_MASK existed only in the
# experiment (reverted, profiles/r02_experiments.json pair_masks_64M): kept as the record of what was run
for m in 0 1; do
  SPHG_PAIR_MASK=$m timeout 900 python bench.py --steps 30 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_mask_$m.log 2>&1
  tail -1 gpurun_out/ab_mask_$m.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('mask=$m', d['ms_per_step'], {k: round(v,2) for k,v in d['stage_ms'].items()})"
done
timeout 900 python -m pytest tests/test_gpu_decomposition.py -q -x -p no:cacheprovider > gpurun_out/ab_dec.log 2>&1; tail -3 gpurun_out/ab_dec.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --deselect tests/test_gpu_decomposition.py > gpurun_out/ab_pytest.log 2>&1; tail -4 gpurun_out/ab_pytest.log
echo done
