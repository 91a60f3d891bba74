#!/bin/bash
# Moves/s vs N (BASELINE metric): bench.py per config, CPU reference on the same moves.
O=gpurun_out/$1; mkdir -p $O; : > $O/vs_n.jsonl
run() { timeout 600 python bench.py --steps 3 --warmup 3 "$@" 2>$O/err.log | grep '^{' >> $O/vs_n.jsonl; }
run --n0 2048 --mu -2 --moves-per-step 1048576
run --n0 2048 --mu 1 --moves-per-step 1048576
run --n0 32768 --mu 1
run --n0 32768 --mu 1 --strategy cell_list
run --n0 32768 --mu 1 --strategy all_pairs --moves-per-step 65536
run --n0 65536 --mu 1
run --n0 262144 --mu 1
run --n0 262144 --mu 1 --strategy cell_list
wc -l $O/vs_n.jsonl
