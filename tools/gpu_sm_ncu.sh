#!/bin/bash
# ncu --set full of one k_engine_sm launch (64k, mu = -3, after a warm-up).
mkdir -p gpurun_out/${1:-smncu}
O=gpurun_out/${1:-smncu}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_engine_sm -s 1 -c 1 \
  -o $O/sm python tools/sm_sweep.py --mode 2 --k 1 --reps 1 --warm 100000 --moves 30000 > $O/ncu.log 2>&1
ncu -i $O/sm.ncu-rep --page source --csv --print-source cuda > $O/source.csv 2>/dev/null
ncu -i $O/sm.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
tail -3 $O/ncu.log; ls -la $O
