timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/h_pytest.log 2>&1
python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
