timeout 900 python -m pytest tests/test_gpu_api.py -q > gpurun_out/g_pytest.log 2>&1
python tools/_debug_step.py > gpurun_out/g_debug.txt 2>&1
V=paper_2604_13880_b200/_variants
export BENCH_ARGS="--field float64"
bash tools/ab.sh 2 $V/base.so $V/old.so > gpurun_out/g_ab.txt 2>&1
