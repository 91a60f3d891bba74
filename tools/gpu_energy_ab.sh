#!/bin/bash
# Full-system energy A/B: packed-FP32 prefilter (default) vs the scalar one
# (GCMC_ENERGY_SCALAR in a -DGCMC_EXPERIMENTS build); energy parity tests.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "energy" 2>&1 | tail -1
timeout 300 python tools/time_energy.py --bf-max 262144 2>&1
GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_scal.so GCMC_ENERGY_SCALAR=1 timeout 300 python tools/time_energy.py --bf-max 0 2>&1
