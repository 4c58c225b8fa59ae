#!/bin/bash
# GPU iteration loop: parity tests, a short bench, and the per-kernel launch list of one step.
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -${TAIL:-5}
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b.log 2>&1 || tail -20 gpurun_out/b.log
python -c "
import json;d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['stage_ms'], d['roofline']['frac'], d['e2e']['ms_per_step'])"
timeout 300 ncu --profile-from-start off --clock-control none --kernel-name-base demangled --metrics gpu__time_duration.sum --csv \
    --log-file gpurun_out/launches_step.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step > /dev/null 2>&1
