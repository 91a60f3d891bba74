O=gpurun_out/r02af; mkdir -p $O
GCMC_ENGINE_PROFILE=1 GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_prof.so timeout 300 python tools/prof_engine.py --n0 1048576 --mu 1 --moves 1048576 --warm 12582912 > $O/phase_1m.log 2>&1
GCMC_ENGINE_PROFILE=1 GCMC_LIB=$PWD/paper_1408_3764_b200/libgcmc_b200_prof.so timeout 300 python tools/prof_engine.py --n0 65536 --mu -3 --moves 1048576 --warm 4194304 --ctas 23 > $O/phase_sweep.log 2>&1
