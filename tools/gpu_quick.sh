#!/bin/bash
# Quick GPU iteration: optional parity tests, a short bench, the ncu launch list.  Run from anywhere.
# usage: tools/gpu_quick.sh <tag> [tests]
cd /root/repo
TAG=${1:-quick}
CMD='A="python bench.py --steps 32 --warmup 3 --no-cpu --e2e-steps 8"; '
if [ "$2" = "tests" ]; then CMD+='timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -4; '; fi
CMD+='timeout 300 $A > gpurun_out/plain.log 2>&1; head -c 200 gpurun_out/plain.log; echo; ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 150 -c 80 --csv --log-file gpurun_out/launches.csv $A > gpurun_out/ncu.log 2>&1; echo ncu rc=$?'
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1500 -- "$CMD" > gpurun_out/call_$TAG.txt 2>&1
grep -vE "^\[gpurun\] (sending|merged)" gpurun_out/call_$TAG.txt | tail -6 | cut -c1-300
python tools/summarize_profiles.py $TAG gpurun_out/launches.csv | sed -n 5,20p
