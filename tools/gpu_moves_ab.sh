#!/bin/bash
# A/B of moves per round (GCMC_E2_MOVES builds) x evaluator group size at the
# bench window, plus the trajectory-identity tests on each variant.
O=gpurun_out/$1; mkdir -p $O
for cfg in "default 256" "default 128" "m384 128" "m512 128"; do
  set -- $cfg
  L=""; [ "$1" != default ] && L="GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_$1.so"
  echo "== lib $1 group $2" >> $O/ab.log
  env $L GCMC_ENGINE_GROUP=$2 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 2>&1 | grep -E "ctas|rror" | tail -3 >> $O/ab.log
done
for cfg in "m512 128" "m384 128"; do
  set -- $cfg
  echo "== tests lib $1 group $2" >> $O/ab.log
  env GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_$1.so GCMC_ENGINE_GROUP=$2 timeout 600 python -m pytest tests -m gpu -q -x -k "1e5 or chunk or drift or checkpoint or ideal or draw" 2>&1 | tail -3 >> $O/ab.log
done
cat $O/ab.log
