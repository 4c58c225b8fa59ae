#!/bin/bash
# Thread-count / FP64-deferral sweep of the cluster Cholesky-inverse (w = 230, 26 factors, FP32 and FP64).
mkdir -p gpurun_out
for T in 192 256; do for D in 0 1; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRKFAC_CC_THREADS=$T -DRKFAC_CC_DEFER64=$D \
       tools/chol_bench.cu -o gpurun_out/cb || exit 1
  echo "T=$T D=$D $(timeout 60 gpurun_out/cb 230 26 0 | head -1) | $(timeout 60 gpurun_out/cb 230 26 1 | head -1) | $(timeout 60 gpurun_out/cb 230 26 1 | grep 'factor 0')"
done; done
