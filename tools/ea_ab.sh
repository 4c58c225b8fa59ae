#!/bin/bash
# A/B of the EA configuration's Cin ring depth (RKFAC_EA_CIN_RING 3 vs 4): EA stage time and HBM fraction, twice each.
mkdir -p gpurun_out
show() { python -c "
import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);print('$2', 'ea_ms %.4f'%d['stage_ms']['ea'], 'frac %.4f'%d['ea_hbm']['frac'], 'step %.3f'%d['ms_per_step'], 'e2e %.3f'%d['e2e']['ms_per_step'])"; }
for R in ${RINGS:-3 4}; do
  rm -f paper_2206_15397_b200/build/tc_gemm.o
  RKFAC_NVCC_DEFS="-DRKFAC_EA_CIN_RING=$R" python -m paper_2206_15397_b200.build > gpurun_out/build_$R.log 2>&1 || { tail gpurun_out/build_$R.log; exit 1; }
  for i in 1 2; do
    timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$R.log 2>&1 || tail -5 gpurun_out/ab_$R.log
    show gpurun_out/ab_$R.log "ring=$R"
  done
done
