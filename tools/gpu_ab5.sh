#!/bin/bash
# GPU suite on the default build, then default vs the HEAD build (libgcmc_b200_head.so)
# at the bench window, interleaved twice.
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1
tail -2 $O/gpu_tests.log > $O/ab.log
for rep in 1 2; do
for lib in head default; do
  L=""; [ "$lib" != default ] && L="GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_$lib.so"
  echo "== lib $lib" >> $O/ab.log
  env $L timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 2>&1 | grep -E "ctas|rror" | tail -3 >> $O/ab.log
done
done
cat $O/ab.log
