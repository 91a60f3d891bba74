#!/bin/bash
O=gpurun_out/${1:-ap}; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_engine_parity.py tests/test_gpu_parity.py -m gpu -q -k "all_pairs or pair_eval" --timeout 900 > $O/ap_tests.log 2>&1
timeout 600 python bench.py --n0 32768 --mu 1 --strategy all_pairs --moves-per-step 262144 --steps 3 --warmup 3 > $O/bench_ap32k.log 2>&1
timeout 600 python bench.py --n0 32768 --mu 1 --strategy microcell --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_mc32k.log 2>&1
