#!/bin/bash
# register / spill report of the hq_v3.cu kernels (development helper)
cd "$(dirname "$0")/../paper_2603_03019_b200/csrc" && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xptxas -v -c hq_v3.cu -o /tmp/hq_v3.o 2>&1 | grep -E "error|Compiling entry|spill|Used" | \
  sed -e 's/ptxas info    : //' | paste - - - | sed -E 's/Compiling entry function .(_ZN3hq3[0-9a-z_]*[^ ]*). for .sm_100a.//' | cut -c1-200
