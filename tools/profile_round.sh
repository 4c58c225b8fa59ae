#!/bin/bash
# Round-end evidence on one GPU (run under gpurun from the repo root):
#   1. the default bench line (with the CPU reference baseline) and the reference arm -> gpurun_out/bench.json, ref.json
#   2. the per-kernel launch list of one step (ncu, time only)                        -> gpurun_out/launches_step.csv
#   3. ncu --set full of the first grouped X*Q, the EA update, one Cholesky-inverse and one tridiagonalisation,
#      each from a single-plan step (--groups 1: deterministic launch order)            -> gpurun_out/*_full.ncu-rep
# Every ncu command profiles `bench.py --profile-step`, which is first run without ncu.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log > gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.log 2>&1; tail -1 gpurun_out/ref.log > gpurun_out/ref.json
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step"
timeout 300 $P > gpurun_out/plain.log 2>&1 || { echo "plain profile-step run failed"; exit 1; }
NCU="ncu --profile-from-start off --clock-control none --kernel-name-base demangled"
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_step.csv $P > /dev/null 2>&1
P1="$P --groups 1"
timeout 300 $P1 > gpurun_out/plain1.log 2>&1 || { echo "plain single-plan profile-step run failed"; exit 1; }
timeout 900 $NCU --set full --import-source on -k regex:tc_gemm_kernel --launch-skip 1 -c 1 -o gpurun_out/xq_full $P1 \
    > gpurun_out/xq_full.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:tc_gemm_kernel --launch-skip 0 -c 1 -o gpurun_out/ea_full $P1 \
    > gpurun_out/ea_full.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:cholinv_cluster --launch-skip 1 -c 1 -o gpurun_out/chol_full $P1 \
    > gpurun_out/chol_full.log 2>&1
timeout 900 $NCU --set full --import-source on -k regex:tridiag1b -c 1 -o gpurun_out/tri_full $P1 \
    > gpurun_out/tri_full.log 2>&1
for k in xq ea chol tri; do python tools/ncu_summary.py gpurun_out/${k}_full.ncu-rep $k > gpurun_out/${k}_full.txt; done
python tools/launches.py gpurun_out/launches_step.csv > gpurun_out/launches_step.txt
rm -f gpurun_out/*.ncu-rep gpurun_out/eig_bench* gpurun_out/chol_bench gpurun_out/tc_acc gpurun_out/eb  # keep the merge under 64 MiB
ls -la gpurun_out
