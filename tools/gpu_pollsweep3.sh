#!/bin/bash
# Sequencer / evaluator poll back-off sweep at the bench window (default engine shape).
O=gpurun_out/$1; mkdir -p $O; : > $O/sweep.log
for cfg in "64 64" "0 0" "32 32" "128 128" "64 0" "0 64" "256 64" "64 256"; do
  set -- $cfg
  echo "== seq $1 eval $2" >> $O/sweep.log
  GCMC_POLL_NS=$1 GCMC_EPOLL_NS=$2 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 2>&1 | grep ctas= >> $O/sweep.log
done
cat $O/sweep.log
