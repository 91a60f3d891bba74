#!/bin/bash
# Chain-per-SM engine A/B of library variants (tools/build_variant.py NAME
# -D...; GCMC_LIB): one chain alone (with GCMC_SM_PHASES role cycles; a
# -DGCMC_SM_STEPS variant adds step cycles) and 148 chains in one launch.
#   VARIANTS="name1 name2" bash tools/gpu_sm_ab.sh
for v in "" $VARIANTS; do
  L=$PWD/paper_1408_3764_b200/libgcmc_b200${v:+_$v}.so
  echo "== ${v:-default}"
  GCMC_LIB=$L GCMC_SM_PHASES=1 timeout 300 python tools/sm_sweep.py --mode 2 --k 1 --reps 1 2>&1 | grep "engine_sm\]" | tail -2
  GCMC_LIB=$L timeout 300 python tools/sm_sweep.py --mode 2 --k 1 148 2>&1 | tail -2 | cut -c1-120
done
