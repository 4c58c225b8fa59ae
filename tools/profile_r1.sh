#!/bin/bash
# One-GPU profiling pass of the VGG16 step (run under gpurun from the repo root). Every ncu command profiles the
# same `bench.py --profile-step` program, which has exited 0 without ncu first.
set -x
OUT=gpurun_out
mkdir -p $OUT
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step"
$P > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
NCU="ncu --profile-from-start off --clock-control none --kernel-name-base demangled"
$NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_step.csv $P > /dev/null 2>&1
$NCU --set full --import-source on -k regex:tc_gemm_kernel -c 2 -o $OUT/tc_ea_xq $P > $OUT/ncu_tc.log 2>&1
$NCU --set full --import-source on -k regex:"grouped_gemm|tdeig|tridiag|cholinv|backxform" -c 6 -o $OUT/latency $P > $OUT/ncu_lat.log 2>&1
ls -la $OUT
