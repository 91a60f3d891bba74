#!/bin/bash
# Full-system energy: parity tests and timing (library variants via VARIANTS="name ...").
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "energy" 2>&1 | tail -1
timeout 300 python tools/time_energy.py --bf-max 262144 2>&1
for v in $VARIANTS; do echo "== $v"; GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_$v.so timeout 300 python tools/time_energy.py --bf-max 0 2>&1; done
