#!/bin/bash
# Round-end style validation: GPU tests, smoke, bench (both arms), the
# launch list, ncu --set full of k_engine2 in the bench window and of
# k_energy, summarised into JSON (profiles/engine_ncu.json, energy_ncu.json);
# the 148-chain sweep bench line and ncu of one k_engine_sm launch.
# usage: bash tools/gpu_final.sh TAG
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
lscpu | grep -E 'Model name|^CPU\(s\)' > $O/lscpu.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout-method=thread --durations=20 > $O/gpu_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.log 2>&1
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
timeout 900 python bench.py --sweep --chains-per-gpu 148 --steps 3 --warmup 3 --no-energy > $O/bench_sweep148.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_engine_sm -s 1 -c 1 -o $O/engine_sm_full \
  python tools/sm_sweep.py --mode 2 --k 148 --reps 1 --warm 200000 --moves 100000 > $O/ncu_sm.log 2>&1
python tools/ncu_engine_sm.py $O/engine_sm_full.ncu-rep $O 14800000 \
  "one launch of the 148-chain 64k sweep (100000 moves per chain after 200000 warm-up moves, mu = -3 + c / 148)" \
  > $O/engine_sm_ncu.json 2> $O/engine_sm_ncu.err
echo done
