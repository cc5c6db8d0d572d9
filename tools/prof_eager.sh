#!/bin/bash
# ncu launch list (graph launches) + --set full of one eager launch of each iteration kernel.
# usage: tools/prof_eager.sh <tag> <field> [extra bench args]   (runs on the GPU box via gpurun)
TAG=$1; FIELD=${2:-float64}; shift 2
A="python bench.py --steps 32 --warmup 3 --no-cpu --e2e-steps 8 --field $FIELD $*"
CMD="$A > gpurun_out/${TAG}_plain.json 2>&1; ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 150 -c 96 --csv --log-file gpurun_out/${TAG}_launches.csv $A > gpurun_out/${TAG}_ncu.log 2>&1; DET_PROFILE_RANGE=1 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'k_sat|k_region|k_row|k_ctrl' -c 6 -o gpurun_out/${TAG}_full $A > gpurun_out/${TAG}_ncufull.log 2>&1; echo done"
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1200 -- "$CMD" > gpurun_out/call_$TAG.txt 2>&1
tail -2 gpurun_out/call_$TAG.txt
python -c "import json;d=json.load(open('gpurun_out/${TAG}_plain.json'));print(d['value'],d['roofline']['phase_ms_per_iteration'])"
python tools/summarize_profiles.py $TAG gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_full.ncu-rep > gpurun_out/${TAG}_summary.md
head -14 gpurun_out/${TAG}_summary.md
