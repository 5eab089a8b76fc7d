#!/bin/bash
# Build libhq.so with ptxas statistics for the sweep kernel (development helper).
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -Xptxas -v \
  -o paper_2603_03019_b200/libhq.so paper_2603_03019_b200/csrc/hq_api.cu paper_2603_03019_b200/csrc/hq_kernels.cu \
  paper_2603_03019_b200/csrc/hq_v2.cu 2>&1 | grep -E "error|warning|k_sweep2" -A3 | grep -E "error|warning|Function prop|registers|spill"
