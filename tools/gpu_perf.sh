#!/bin/bash
# Engine performance check: 1M (prof_engine), 64k sweep K=6, phase profile of one 64k chain, parity.
O=gpurun_out/${1:-perf}; mkdir -p $O
timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 4194304 --warm 12582912 > $O/1m.log 2>&1
echo "1M: $(tail -1 $O/1m.log)" >> $O/summary.txt
timeout 600 python bench.py --sweep --chains-per-gpu 6 --steps 3 --warmup 3 --no-cpu-baseline --no-energy > $O/sweep6.log 2>&1
python -c "
import json; l=json.loads(open('$O/sweep6.log').read().strip().splitlines()[-1])
print('sweep K=6', 'value %.4g'%l['value'], 'mpr %.1f'%l['moves_per_round'], 'nspr %.0f'%l['ns_per_round'])" >> $O/summary.txt
GCMC_ENGINE_PROFILE=1 GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_prof.so timeout 300 python tools/prof_engine.py --n0 65536 --mu -3 --moves 1048576 --warm 4194304 --ctas 23 > $O/phase_sweep.log 2>&1
GCMC_ENGINE_PROFILE=1 GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_prof.so timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 1048576 --warm 12582912 > $O/phase_1m.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_engine_parity.py tests/test_gpu_chains.py tests/test_gpu_parity.py -m gpu -q --timeout 600 > $O/parity.log 2>&1
tail -1 $O/parity.log >> $O/summary.txt
