#!/bin/bash
O=gpurun_out/$1; mkdir -p $O
for cfg in "0 0" "64 64" "0 500" "0 2000" "500 0" "200 200"; do
  set -- $cfg
  echo "== seq $1 eval $2" >> $O/sweep.log
  GCMC_POLL_NS=$1 GCMC_EPOLL_NS=$2 timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 262144 --warm 262144 2>&1 | grep ctas >> $O/sweep.log
done
