#!/bin/bash
# Rows-per-chunk (U) sweep of the one-barrier tridiagonalisation on 26 cores of w = 230 (eigensolver total).
mkdir -p gpurun_out
for U in 1 2 1 2; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRKFAC_T1B_U=$U \
       tools/eig_bench.cu paper_2206_15397_b200/csrc/misc.cu -o gpurun_out/eb || exit 1
  echo "U=$U $(timeout 60 gpurun_out/eb 230 26 | head -1)"
done
