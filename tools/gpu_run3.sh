# D2 + combined prime-path/head queue: count-mode parity and the config-5 bench (3 runs)
python -m pytest tests/test_gpu_count.py tests/test_gpu_boundaries.py -q -x > gpurun_out/pytest_count3.log 2>&1; echo PYTEST_EXIT=$? >> gpurun_out/pytest_count3.log
for i in 1 2; do python bench.py --no-cpu-baseline --no-secondary --no-e2e > gpurun_out/bench3_$i.log 2>&1; done
