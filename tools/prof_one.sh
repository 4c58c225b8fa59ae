#!/bin/bash
# ncu --set full of the N-th launch of a kernel in one VGG16 step: bash tools/prof_one.sh <regex> <skip> <name>
mkdir -p gpurun_out
P="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step"
$P > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain.log; exit 1; }
ncu --profile-from-start off --clock-control none --kernel-name-base demangled --set full --import-source on \
    -k "regex:$1" --launch-skip "$2" -c 1 -o "gpurun_out/$3" $P > "gpurun_out/$3.log" 2>&1
tail -2 "gpurun_out/$3.log"
