#!/bin/bash
# ncu --set full (with source) of one k_energy_pk launch at 1M; source-line CSV.
mkdir -p gpurun_out/${1:-enncu}; O=gpurun_out/${1:-enncu}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_energy_pk -c 1 -o $O/en \
  python tools/time_energy.py --bf-max 0 --sizes 1048576 > $O/ncu.log 2>&1
ncu -i $O/en.ncu-rep --page source --csv --print-source cuda,sass > $O/src.csv 2>/dev/null
ncu -i $O/en.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
tail -2 $O/ncu.log
