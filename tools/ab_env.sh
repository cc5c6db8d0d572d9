#!/bin/bash
# A/B device throughput of environment settings on one box, interleaved:
#   tools/ab_env.sh <rounds> "<ENV=V ...>" "<ENV=V ...>" ...   (prints one "setting value" line per run)
R=$1; shift
for i in $(seq $R); do
  for E in "$@"; do
    v=$(env $E timeout 300 python bench.py --steps 64 --warmup 8 --no-cpu --no-extra --e2e-steps 16 $BENCH_ARGS 2>/dev/null | python -c 'import sys,json; print(round(json.loads(sys.stdin.read().strip().splitlines()[-1])["value"]))')
    echo "$E $v"
  done
done
