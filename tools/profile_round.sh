#!/bin/bash
# Round-end evidence on one GPU (run under gpurun from the repo root):
#   1. the default bench line (with the CPU reference baseline)         -> gpurun_out/bench.json
#   2. the per-kernel launch list of one step (ncu, time only)          -> gpurun_out/launches_step.csv
#   3. ncu --set full of the dominant kernel (the first grouped X*Q)    -> gpurun_out/xq_full.ncu-rep
#   4. ncu --set full of the EA update (HBM-bound stage)                -> gpurun_out/ea_full.ncu-rep
# Every ncu command profiles `bench.py --profile-step`, which is first run without ncu.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step"
timeout 300 $P > gpurun_out/plain.log 2>&1 || { echo "plain profile-step run failed"; exit 1; }
NCU="ncu --profile-from-start off --clock-control none --kernel-name-base demangled"
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_step.csv $P > /dev/null 2>&1
timeout 900 $NCU --set full --import-source on -k regex:tc_gemm_kernel --launch-skip 1 -c 1 -o gpurun_out/xq_full $P \
    > gpurun_out/xq_full.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:tc_gemm_kernel --launch-skip 0 -c 1 -o gpurun_out/ea_full $P \
    > gpurun_out/ea_full.log 2>&1
ls -la gpurun_out
