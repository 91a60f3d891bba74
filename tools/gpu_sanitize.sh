#!/bin/bash
O=gpurun_out/${1:-sanitize}; mkdir -p $O
for t in memcheck racecheck synccheck; do
  MOVES=${MOVES:-4000} timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > $O/$t.log 2>&1
  echo "$t rc=$?" >> $O/summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|========= [0-9]+ errors|Invalid|Race|hazard" $O/$t.log | tail -5 >> $O/summary.txt
done
