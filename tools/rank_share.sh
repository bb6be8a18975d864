for n in 2 4 8; do timeout 900 python tools/rank_share.py $n 20 > gpurun_out/rs_$n.log 2>&1; tail -1 gpurun_out/rs_$n.log; done
