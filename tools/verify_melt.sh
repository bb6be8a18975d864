timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/melt_l_a.csv python tools/melt_steps.py > gpurun_out/melt_ncu_a.log 2>&1
SPHG_REPART_ALL=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/melt_l_b.csv python tools/melt_steps.py > gpurun_out/melt_ncu_b.log 2>&1
echo done
