#!/bin/bash
# Per-kernel eager durations (ncu gpu__time_duration, serialised) of the bench's kernel_times pass,
# one CSV per setting: tools/kt_ncu.sh <tag> "<ENV=V ...>" ...
TAG=$1; shift
i=0
for E in "$@"; do
  env $E DET_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_ --csv \
    --log-file gpurun_out/${TAG}_kt$i.csv python bench.py --steps 8 --warmup 3 --no-cpu --no-extra --e2e-steps 4 > /dev/null 2>&1
  echo "$E -> gpurun_out/${TAG}_kt$i.csv rc=$?"
  i=$((i+1))
done
