#!/bin/bash
# A/B of the EA operand lo planes: formed in smem by the converter warps (default) vs stored by a split pass
# (RKFAC_EA_STORED_LO=1), on VGG16 (n = 128) and config 5 (n = 512).
mkdir -p gpurun_out
for w in vgg16 wide16384; do for L in 0 1; do
  RKFAC_EA_STORED_LO=$L timeout 400 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/lo_$w$L.log 2>&1 || tail -3 gpurun_out/lo_$w$L.log
  python -c "
import json;d=json.loads(open('gpurun_out/lo_$w$L.log').read().strip().splitlines()[-1]);print('$w stored_lo=$L', 'ea_ms %.4f'%d['stage_ms']['ea'], 'step %.3f'%d['ms_per_step'], 'e2e %.3f'%d['e2e']['ms_per_step'])"
done; done
RKFAC_EA_STORED_LO=1 timeout 300 python -m pytest tests -m gpu -x -q -k "ea or step" 2>&1 | tail -1
