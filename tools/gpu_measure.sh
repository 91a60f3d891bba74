#!/bin/bash
# Measurement pass on one B200: ubench (latency floor inputs), bench.py
# (1M default; the 64k sweep with K chains per GPU), moves/s vs N, the launch
# list, and one ncu --set full capture of k_engine2 in the bench window
# (after 5 warm-up steps of 2^22 moves: the 11th engine launch), summarised.
# usage: bash tools/gpu_measure.sh TAG [skip-sweep]
TAG=${1:-measure}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
lscpu | grep -E 'Model name|^CPU\(s\)' > $O/lscpu.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -I paper_1408_3764_b200/csrc \
     -I include -o /tmp/ubench tools/ubench/ubench.cu > /dev/null 2>&1
timeout 120 /tmp/ubench > $O/ubench.txt 2>&1
timeout 120 /tmp/ubench --json 2> $O/ubench.json > /dev/null
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.log 2>&1
if [ -z "$2" ]; then
  for K in 1 2 4 6 8; do
    timeout 900 python bench.py --sweep --chains-per-gpu $K --steps 3 --warmup 3 > $O/sweep_k$K.log 2>&1
  done
  bash tools/gpu_vs_n.sh $TAG
fi
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-energy > $O/ncu_launch_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_engine2 -s 10 -c 1 \
  -o $O/engine2_full python bench.py --steps 1 --warmup 5 --no-cpu-baseline --no-energy > $O/ncu_full.log 2>&1
python tools/ncu_engine.py $O/engine2_full.ncu-rep 2097152 $O \
  "one launch of 2^21 moves at 1M, mu=+1 (bench.py --steps 1 --warmup 5: the 11th k_engine2 launch, moves 20.97M..23.07M, inside the bench window), ncu --set full --clock-control none" \
  > $O/engine_ncu.json 2> $O/engine_ncu.err
timeout 900 ncu --set full --clock-control none -k regex:k_energy -c 1 -o $O/energy_full \
  python tools/time_energy.py --bf-max 0 --sizes 1048576 > $O/ncu_energy.log 2>&1
python tools/ncu_energy.py $O/energy_full.ncu-rep $O > $O/energy_ncu.json 2> $O/energy_ncu.err
echo done
