#!/bin/bash
# Round-2 evidence on one GPU (run under gpurun from the repo root), VERDICT r01 missing #8 / #9:
#   1. ncu --set full of the kernels not yet captured, each from one single-plan VGG16 step (--groups 1):
#      the four apply-stage tc_gemm launches (the last four tc_gemm launches of the step), the FP64 DMMA Gram and
#      triangular product, bisection, eigenvectors, back-transformation, Omega            -> gpurun_out/*_full.txt
#   2. compute-sanitizer memcheck / racecheck / synccheck over the smoke step and memcheck over a slice of the GPU
#      parity tests                                                                          -> gpurun_out/sanitizer_*.log
set -u
mkdir -p gpurun_out
P1="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --profile-step --groups 1"
timeout 300 $P1 > gpurun_out/plain1.log 2>&1 || { echo "plain single-plan profile-step run failed"; exit 1; }
NCU="ncu --profile-from-start off --clock-control none --kernel-name-base demangled --set full --import-source on"
# tc_gemm launches of one step: EA 1, decomposition 30 (9 power products, 16 + 2 CholeskyQR GEMMs, final product,
# core, lift), then the 4 apply GEMMs
timeout 900 $NCU -k regex:tc_gemm_kernel --launch-skip 31 -c 4 -o gpurun_out/apply_full $P1 > gpurun_out/apply_full.log 2>&1
for spec in "gram64:gram64_kernel" "tri64:tri64_kernel" "bisect:bisect_kernel" "eigvec:eigvec_kernel" \
            "backxform:backxform_wy_kernel" "omega:omega_kernel" "split:split_kernel"; do
  name=${spec%%:*}; kern=${spec#*:}
  timeout 600 $NCU -k regex:$kern -c 1 -o gpurun_out/${name}_full $P1 > gpurun_out/${name}_full.log 2>&1
done
for k in apply gram64 tri64 bisect eigvec backxform omega split; do
  python tools/ncu_summary.py gpurun_out/${k}_full.ncu-rep $k > gpurun_out/${k}_full.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
# compute-sanitizer: refused on this GPU pool ("closed ... runs under it have left GPUs needing a reset", exit 86;
# profiles/r02_compute_sanitizer_refused.txt); the commands stay for pools that allow it
if [ "${RKFAC_RUN_SANITIZER:-0}" = "1" ]; then
CS="compute-sanitizer --error-exitcode 9 --print-limit 20"
timeout 900 $CS --tool memcheck python __graft_entry__.py smoke > gpurun_out/sanitizer_memcheck_smoke.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer_memcheck_smoke.log
timeout 900 $CS --tool racecheck python __graft_entry__.py smoke > gpurun_out/sanitizer_racecheck_smoke.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer_racecheck_smoke.log
timeout 900 $CS --tool synccheck python __graft_entry__.py smoke > gpurun_out/sanitizer_synccheck_smoke.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer_synccheck_smoke.log
timeout 1200 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -q -x \
    -k "config1 or apply or ea_update or batched_step_matches or single_factor or nccl or gather" \
    > gpurun_out/sanitizer_memcheck_tests.log 2>&1
echo "exit $?" >> gpurun_out/sanitizer_memcheck_tests.log
fi
ls -la gpurun_out | tail -30
