#!/bin/bash
# One gpurun call: plain bench line, ncu launch list of the TIMED graph launches (DET_PROFILE_RANGE=2),
# and ncu --set full of one eager launch of each iteration kernel (DET_PROFILE_RANGE=1).
# usage (on the GPU box): bash tools/prof_r02.sh <tag> [extra bench args]
TAG=$1; shift
A="python bench.py --steps 16 --warmup 3 --no-cpu --e2e-steps 8 $*"
python bench.py $* > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
DET_PROFILE_RANGE=2 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -c 768 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $A > gpurun_out/${TAG}_ncu.log 2>&1
DET_PROFILE_RANGE=1 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:'k_sat|k_region|k_row|k_ctrl|k_advect' -c 7 -o gpurun_out/${TAG}_full $A > gpurun_out/${TAG}_ncufull.log 2>&1
echo done
