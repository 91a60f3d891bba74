#!/bin/bash
# Full GPU suite on the 384-move / 128-thread-group shape, then an A/B of the
# moves per round at the bench window (interleaved, twice).
O=gpurun_out/$1; mkdir -p $O
GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_m384.so GCMC_ENGINE_GROUP=128 timeout 900 python -m pytest tests -m gpu -q -x > $O/gpu_tests_m384.log 2>&1
tail -2 $O/gpu_tests_m384.log > $O/ab.log
for rep in 1 2; do
for cfg in "default 256" "m320 128" "m384 128"; do
  set -- $cfg
  L=""; [ "$1" != default ] && L="GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_$1.so"
  echo "== lib $1 group $2" >> $O/ab.log
  env $L GCMC_ENGINE_GROUP=$2 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 2>&1 | grep -E "ctas|rror" | tail -3 >> $O/ab.log
done
done
cat $O/ab.log
