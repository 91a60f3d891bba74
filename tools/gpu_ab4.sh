#!/bin/bash
# GPU suite on the default build, moves-per-round A/B at the bench window,
# phase profile of the default shape.
O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/gpu_tests.log 2>&1
tail -2 $O/gpu_tests.log > $O/ab.log
for rep in 1 2; do
for cfg in "default 128" "m512 128"; do
  set -- $cfg
  L=""; [ "$1" != default ] && L="GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_$1.so"
  echo "== lib $1 group $2" >> $O/ab.log
  env $L GCMC_ENGINE_GROUP=$2 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 2>&1 | grep -E "ctas|rror" | tail -3 >> $O/ab.log
done
done
env GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_prof384.so GCMC_ENGINE_PROFILE=1 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 1048576 --warm 12582912 2>&1 | grep -v "^\[round\|eupd" | tail -14 > $O/prof.log
cat $O/ab.log
