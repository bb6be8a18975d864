bash tools/prof_round.sh r02
bash tools/prof_build64.sh r02
ls -la gpurun_out/
