timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "channels or field or golden or trajectory or engine" > gpurun_out/j_pytest.log 2>&1
V=paper_2604_13880_b200/_variants
export BENCH_ARGS="--field float64"
bash tools/ab.sh 3 $V/base.so $V/quad2.so > gpurun_out/j_ab.txt 2>&1
