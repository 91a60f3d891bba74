#!/bin/bash
# A/B of engine2 variants (GCMC_E2_VARIANT bits) on one box, 1M mu=+1, bench window.
O=gpurun_out/${1:-variants}; mkdir -p $O; shift
for v in "$@"; do
  GCMC_E2_VARIANT=$v timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 > $O/variant$v.log 2>&1
  echo "variant $v: $(tail -1 $O/variant$v.log)" >> $O/summary.txt
done
