#!/bin/bash
# Phase-timer profile of the default engine shape at the bench window
# (needs: python tools/build_variant.py prof -DGCMC_PHASE_TIMERS -DGCMC_EXPERIMENTS).
# usage: bash tools/gpu_phase.sh TAG [extra env assignments...]
O=gpurun_out/$1; mkdir -p $O; shift
for rep in 1; do
  env "$@" GCMC_WALK_REPS=$rep GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_prof.so GCMC_ENGINE_PROFILE=1 \
    timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 1048576 --warm 12582912 2>&1 \
    | grep -v "^\[round\|eupd" | tail -16 > $O/phase_reps$rep.log
done
