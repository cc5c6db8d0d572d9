#!/bin/bash
# A/B device throughput of library builds on one box, interleaved: tools/ab.sh <rounds> <lib.so>...
# (DET_LIB selects the build; prints one "lib value" line per run)
R=$1; shift
for i in $(seq $R); do
  for L in "$@"; do
    v=$(DET_LIB=$L timeout 300 python bench.py --steps 64 --warmup 8 --no-cpu --no-extra --e2e-steps 16 $BENCH_ARGS 2>/dev/null | python -c 'import sys,json; print(round(json.loads(sys.stdin.read().strip().splitlines()[-1])["value"]))')
    echo "$(basename $L) $v"
  done
done
