S=/usr/local/cuda/bin/compute-sanitizer
for lib in _det.so _variants/old.so; do
  export DET_LIB=paper_2604_13880_b200/$lib
  for tool in memcheck racecheck synccheck; do
    echo "=== $lib $tool" >> gpurun_out/f_san.txt
    timeout 600 $S --tool $tool --print-limit 20 python tools/sanitize_case.py float64 6 >> gpurun_out/f_san.txt 2>&1
  done
done
