#!/bin/bash
# one bench run summarised on one line: bash tools/bline.sh LABEL [bench args...]
L=$1; shift
python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" 2>gpurun_out/bline.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$L', 'step %.3f' % d['ms_per_step'], 'e2e %.3f' % d['e2e']['ms_per_step'], 'xq %.3f' % d['roofline']['frac'], {k: round(v, 3) for k, v in d['stage_ms'].items()})" | tee -a gpurun_out/bline.txt
