#!/bin/bash
# Round-end validation (tools/gpu_final.sh) plus the small-box bench lines.
TAG=${1:-final}
bash tools/gpu_final.sh $TAG
O=gpurun_out/$TAG
for args in "--n0 2048 --mu -2 --moves-per-step 1048576" "--n0 2048 --mu 1 --moves-per-step 1048576" "--n0 32768 --mu 1"; do
  timeout 300 python bench.py --steps 3 --warmup 3 $args 2>/dev/null | grep '^{' >> $O/vs_n_small.jsonl
done
echo done2
