mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DRKFAC_PHASE_TIMING tools/chol_bench.cu -o /tmp/cbp || exit 1
timeout 60 /tmp/cbp 230 26 0 | head -6
timeout 60 /tmp/cbp 230 26 1 | head -6
