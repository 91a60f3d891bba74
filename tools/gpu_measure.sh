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
ncu -i $O/energy_full.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; u=r[1]; d=r[2]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','sm__warps_active.avg.pct_of_peak_sustained_active','lts__t_sector_hit_rate.pct','launch__registers_per_thread']
print('k_energy at 1M (random start, rho 0.67), ncu --set full --clock-control none'); print(); print('| metric | value | unit |'); print('|---|---|---|')
[print('|',m,'|',d[h.index(m)],'|',u[h.index(m)],'|') for m in want if m in h]
" > $O/energy_ncu.md
echo done
