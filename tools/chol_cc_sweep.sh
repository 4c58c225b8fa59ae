#!/bin/bash
# Cluster-size sweep of the cluster Cholesky-inverse (w = 230, 26 factors and 4 factors, FP32 and FP64).
mkdir -p gpurun_out
for C in 2 4 8; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRKFAC_CC_CTAS=$C \
       tools/chol_bench.cu -o gpurun_out/cb$C || exit 1
  echo "C=$C $(timeout 60 gpurun_out/cb$C 230 26 0 | head -1) | $(timeout 60 gpurun_out/cb$C 230 4 0 | head -1) | $(timeout 60 gpurun_out/cb$C 230 26 1 | head -1) | $(timeout 60 gpurun_out/cb$C 230 26 0 | grep 'factor 0')"
done
rm -f gpurun_out/cb?
