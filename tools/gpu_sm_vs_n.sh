#!/bin/bash
# Chain-per-SM engine: 148 replica chains (mu = +1, seeds 1..148) vs N, and one chain alone.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/${1:-smvn}; O=gpurun_out/${1:-smvn}
# warm-up: 64 moves per particle (at least 2M), the equilibrated regime
for n in ${NS:-2048 32768 65536 262144}; do
  W=$(( n * 64 > 2000000 ? n * 64 : 2000000 ))
  timeout 900 python tools/sm_sweep.py --mode 2 --k 1 148 --n0 $n --mu0 1.0 --spread 0 --warm $W --moves ${MOVES:-400000} 2>&1 | tail -2 | sed "s/^/n0=$n warm=$W /" | tee -a $O/vs_n.jsonl
done
