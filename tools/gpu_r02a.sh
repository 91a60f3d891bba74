O=gpurun_out/r02a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_engine_parity.py -m gpu -q -x --durations=15 > $O/gpu_tests_new.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --durations=10 > $O/gpu_tests_old.log 2>&1
echo done
