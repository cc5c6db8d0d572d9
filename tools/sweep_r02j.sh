run() { v=$(env $1 timeout 300 python bench.py --steps 64 --warmup 8 --no-cpu --no-extra --e2e-steps 16 $2 2>/dev/null | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]), d["ms_per_step"], d.get("frames_active_after"))'); echo "$1 | $2 | $v"; }
run X=1 ""
run X=1 "--batch 148"
run DET_WALK_STEPS=12 "--batch 148"
run DET_WALK_STEPS=8 "--batch 148"
run DET_WALK_STEPS=8 "--batch 296"
run DET_WALK_STEPS=8 "--batch 222"
run DET_WALK_STEPS=8 "--batch 148 --groups 4"
