# the GPU suite on the checked build (-DSPHG_CHECKED: rows and index lists validated at every rebuild /
# transition batch; compute-sanitizer is closed on this pool)
SPHG_LIB=libsphg_checked.so timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/checked.log 2>&1; tail -4 gpurun_out/checked.log
