#!/bin/bash
# Multisection width sweep of the Sturm bisection (threads per eigenvalue) on 26 cores of w = 230 (eigensolver total).
mkdir -p gpurun_out
for G in 4 8 16 4 8 16; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRKFAC_BIS_G=$G \
       tools/eig_bench.cu paper_2206_15397_b200/csrc/misc.cu -o gpurun_out/eb || exit 1
  echo "G=$G $(timeout 60 gpurun_out/eb 230 26 | head -2 | tr '\n' ' ')"
done
