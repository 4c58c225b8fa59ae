#!/bin/bash
# A/B of the Cholesky-inverse kernels on VGG16-shaped Gram matrices (cluster vs single CTA), FP32 and FP64.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DRKFAC_PHASE_TIMING tools/chol_bench.cu -o gpurun_out/chol_bench || exit 1
for args in "230 26 0" "230 26 1" "272 4 0" "64 6 0" "100 3 1"; do
  echo "== $args"; timeout 60 gpurun_out/chol_bench $args
  RKFAC_CHOLINV_SINGLE=1 timeout 60 gpurun_out/chol_bench $args | head -1
done
