#!/bin/bash
# Build + run the GEMM debug timeline on the GPU box (cg=1 vs cg=2).
set -e
cd "$(dirname "$0")/.."
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DBC_GEMM_TRACE -Ipaper_2511_20426_b200/csrc -Iinclude \
  scripts/gemm_trace.cu paper_2511_20426_b200/csrc/common.cpp -o /tmp/gemm_trace
/tmp/gemm_trace 1
/tmp/gemm_trace 2
