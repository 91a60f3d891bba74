#!/bin/bash
# ncu launch list of the bench + one full capture of k_engine2 (TAG arg)
TAG=${1:-n}
O=gpurun_out/$TAG
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_engine2 -s 2 -c 1 -o $O/engine2_full python bench.py --steps 1 --warmup 1 --moves-per-step 65536 --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done
