#!/bin/bash
# Chain-per-SM engine: per-chain phase cycles when K chains share the GPU.
mkdir -p gpurun_out/${1:-sm}
O=gpurun_out/${1:-sm}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for K in 1 16; do
GCMC_SM_PHASES=1 timeout 300 python tools/sm_sweep.py --mode 2 --k $K --reps 1 > $O/k$K.jsonl 2> $O/k$K.err
echo "K=$K"; grep engine_sm $O/k$K.err | tail -4; cat $O/k$K.jsonl
done
GCMC_SM_PHASES=1 timeout 300 python tools/sm_sweep.py --mode 2 --k 16 --n0 8192 --reps 1 > $O/k16s.jsonl 2> $O/k16s.err
echo "K=16 n0=8192"; grep engine_sm $O/k16s.err | tail -3; cat $O/k16s.jsonl
GCMC_SM_PHASES=1 timeout 300 python tools/sm_sweep.py --mode 2 --k 1 --n0 8192 --reps 1 > $O/k1s.jsonl 2> $O/k1s.err
echo "K=1 n0=8192"; grep engine_sm $O/k1s.err | tail -2; cat $O/k1s.jsonl
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
