#!/bin/bash
# Register-tile width sweep of the cluster Cholesky-inverse update (w = 230, 26 and 4 factors; FP32 and FP64).
mkdir -p gpurun_out
for TW in 4 8; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRKFAC_CC_TW32=$TW -DRKFAC_CC_TW64=$TW \
       tools/chol_bench.cu -o /tmp/cbt$TW || exit 1
  for F in "230 26 0" "230 4 0" "230 26 1" "200 10 0" "100 7 0" "64 5 1"; do
    echo "TW=$TW $(timeout 60 /tmp/cbt$TW $F | grep -v '^block' | tr '\n' ' ')"
  done
done
