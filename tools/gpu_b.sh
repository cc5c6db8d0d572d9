#!/bin/bash
# one gpurun call: new GPU tests + ncu launch list + --set full of the float64 path (tag $1)
TAG=${1:-r02a}
A="python bench.py --steps 32 --warmup 3 --no-cpu --e2e-steps 8 --field float64"
timeout 600 python -m pytest tests/test_gpu_api.py -x -q > gpurun_out/${TAG}_pytest.log 2>&1
$A > gpurun_out/${TAG}_plain.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 150 -c 96 --csv --log-file gpurun_out/${TAG}_launches.csv $A > gpurun_out/${TAG}_ncu.log 2>&1
DET_PROFILE_RANGE=1 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'k_sat|k_region|k_row|k_ctrl' -c 6 -o gpurun_out/${TAG}_full $A > gpurun_out/${TAG}_ncufull.log 2>&1
echo done
