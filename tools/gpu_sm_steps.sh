#!/bin/bash
# Chain-per-SM engine: step cycles of the diagnostics build (-DGCMC_SM_STEPS).
GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_steps.so GCMC_SM_PHASES=1 timeout 300 python tools/sm_sweep.py --mode 2 --k 1 --reps 1 2>&1 | tail -3
