V=paper_2604_13880_b200/_variants
export BENCH_ARGS="--field float64"
bash tools/ab.sh 3 $V/base.so $V/c2m1.so $V/c2m2.so $V/rw16.so > gpurun_out/i_ab.txt 2>&1
export BENCH_ARGS="--field float64 --groups 4"
bash tools/ab.sh 2 $V/base.so $V/c2m1.so $V/c2m2.so $V/rw16.so >> gpurun_out/i_ab.txt 2>&1
