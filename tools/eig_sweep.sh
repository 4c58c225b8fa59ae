#!/bin/bash
# Variant sweep of the one-barrier tridiagonalisation (threads, rows per chunk, load-first) on 26 cores of w = 230.
mkdir -p gpurun_out
for T in 96 128 192 256; do for U in 1 2; do for LF in 1; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRKFAC_T1B_THREADS=$T -DRKFAC_T1B_U=$U \
       -DRKFAC_T1B_LOADFIRST=$LF tools/eig_bench.cu paper_2206_15397_b200/csrc/misc.cu -o gpurun_out/eb || exit 1
  echo "T=$T U=$U LF=$LF $(timeout 60 gpurun_out/eb 230 26 | head -1)"
done; done; done
RKFAC_TRIDIAG_TWO_BARRIER=1 timeout 60 gpurun_out/eb 230 26 | head -1
