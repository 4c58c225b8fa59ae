#!/bin/bash
# Eigensolver on VGG16-shaped cores: timing, per-phase stamps of steps 10 / 200 of the one-barrier
# tridiagonalisation, and one ncu --set full capture of it.
mkdir -p gpurun_out
for k in 10 200; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -DRKFAC_TRC_TIMING=$k tools/eig_bench.cu \
       paper_2206_15397_b200/csrc/misc.cu -o gpurun_out/eig_bench || exit 1
  timeout 60 gpurun_out/eig_bench 230 26 | head -2
done
timeout 300 ncu --set full --import-source on -k regex:tridiag1b -c 1 -o gpurun_out/tridiag1b gpurun_out/eig_bench 230 26 > gpurun_out/ncu_tri.log 2>&1
tail -2 gpurun_out/ncu_tri.log
