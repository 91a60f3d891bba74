#!/bin/bash
# Chain-per-SM engine A/B of library variants (GCMC_LIB): solo and 148-chain rates.
for v in "" $VARIANTS; do
  L=$PWD/paper_1408_3764_b200/libgcmc_b200${v:+_$v}.so
  echo "== ${v:-default}"
  GCMC_LIB=$L timeout 300 python tools/sm_sweep.py --mode 2 --k 1 148 2>&1 | tail -2 | cut -c1-120
done
