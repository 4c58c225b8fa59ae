#!/bin/bash
# ncu --set full of one CTA-pair X*Q launch (single-plan step): bash tools/prof_pair.sh
mkdir -p gpurun_out
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step --groups 1"
$P > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain.log; exit 1; }
ncu --profile-from-start off --clock-control none --kernel-name-base demangled --set full --import-source on \
    -k "regex:tc_gemm_kernel<.int.${CFG:-3}>" --launch-skip "${SKIP:-2}" -c 1 -o gpurun_out/pairxq $P > gpurun_out/pairxq.log 2>&1
tail -2 gpurun_out/pairxq.log
python tools/ncu_summary.py gpurun_out/pairxq.ncu-rep pairxq | tee gpurun_out/pairxq.txt
ncu -i gpurun_out/pairxq.ncu-rep --page raw --csv > gpurun_out/pairxq_raw.csv
rm -f gpurun_out/pairxq.ncu-rep
