#!/bin/bash
# Build an A/B variant of the library: tools/build_variant.sh <name> [-DFLAG=V ...]
# -> paper_2604_13880_b200/_variants/<name>.so (git-ignored; ships to the GPU box with gpurun)
N=$1; shift
mkdir -p /root/repo/paper_2604_13880_b200/_variants
cd /root/repo/paper_2604_13880_b200/csrc
/usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -cudart static \
  -gencode arch=compute_100a,code=sm_100a -I../../include "$@" -shared -o ../_variants/$N.so det_api.cu
