#!/bin/bash
# A/B of two library builds on one box (1M, prof_engine): usage: bash tools/gpu_libab.sh TAG libA.so libB.so [...]
O=gpurun_out/${1:-libab}; mkdir -p $O; shift
for rep in 1 2; do
  for lib in "$@"; do
    GCMC_LIB=$PWD/$lib timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 > $O/run.log 2>&1
    echo "$lib: $(tail -1 $O/run.log)" >> $O/summary.txt
  done
done
