#!/bin/bash
O=gpurun_out/${1:-misc}; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/init_launches.csv python -c "
import sys; sys.path.insert(0,'.')
from paper_1408_3764_b200 import engine as E
n=262144; box=(n/0.67)**(1/3)
E.random_initial_configuration(n, box, 0.85, 1, device=0)
" > $O/init_ncu.log 2>&1
bash tools/gpu_sanitize.sh ${1:-misc}
