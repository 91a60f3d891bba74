#!/bin/bash
# Source-level stall sampling of one k_engine launch in the bench window.
O=gpurun_out/$1; mkdir -p $O
timeout 900 ncu --section WarpStateStats --section SourceCounters --import-source on --clock-control none \
  -k regex:k_engine --launch-skip 6 --launch-count 1 -o $O/src -f \
  python tools/prof_engine.py --n0 1048576 --mu 1 --moves 2097152 --warm 12582912 > $O/ncu.log 2>&1
tail -3 $O/ncu.log
