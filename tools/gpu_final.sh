#!/bin/bash
# Round-end style validation: GPU tests, smoke, bench (both arms), ncu launch
# list + one full k_engine2 capture. usage: bash tools/gpu_final.sh TAG
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_engine2 -s 2 -c 1 -o $O/engine2_full python bench.py --steps 1 --warmup 1 --moves-per-step 65536 --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done
