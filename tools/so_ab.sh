#!/bin/bash
# A/B of two prebuilt libraries (abso/A.so, abso/B.so; git-ignored): bench stage times, alternating, twice each.
mkdir -p gpurun_out
show() { python -c "
import json;d=json.loads(open('$1').read().strip().splitlines()[-1]);print('$2', 'ea_ms %.4f'%d['stage_ms']['ea'], 'ea_frac %.4f'%d['ea_hbm']['frac'], 'xq_frac %.4f'%d['roofline']['frac'], 'step %.3f'%d['ms_per_step'], 'e2e %.3f'%d['e2e']['ms_per_step'])"; }
for i in 1 2; do for V in A B; do
  cp abso/$V.so paper_2206_15397_b200/librkfac_b200.so
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$V.log 2>&1 || tail -5 gpurun_out/ab_$V.log
  show gpurun_out/ab_$V.log "$V"
done; done
