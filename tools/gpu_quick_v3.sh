#!/bin/bash
# quick engine2 check: smoke, selected parity tests, short bench, phase-timer
# bench (prof variant), delayed-commit drift check (dly variant)
O=gpurun_out/${1:-q}
mkdir -p $O
bash tools/gpu_quick_v2.sh ${1:-q} "$2"
GCMC_LIB=paper_1408_3764_b200/libgcmc_b200_prof.so GCMC_ENGINE_PROFILE=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "engine2 prof|engine prof|dbg\] (after go|latency)" > $O/prof.log
GCMC_LIB=paper_1408_3764_b200/libgcmc_b200_dly.so timeout 300 python tools/debug_first.py 32768 1024 65536 > $O/dly.log 2>&1
