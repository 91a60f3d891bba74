#!/bin/bash
# A/B: bench-window engine profile of the default library and variants.
O=gpurun_out/$1; mkdir -p $O; shift
for lib in default "$@"; do
  L=""; [ "$lib" != default ] && L="GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_$lib.so"
  echo "== $lib" >> $O/ab.log
  env $L GCMC_ENGINE_PROFILE=1 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 2>&1 | grep -E "ctas|sequencer|evaluator|helpers" | tail -4 >> $O/ab.log
done
cat $O/ab.log
