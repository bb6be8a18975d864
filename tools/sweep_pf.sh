for v in pf1 pf0; do
  SPHG_LIB=libsphg_$v.so timeout 600 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pf_$v.log 2>&1
done
echo done
