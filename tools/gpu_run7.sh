# segment phase on the D2 kernel: count + TP count-mode parity (configs 3-5 incl.), bench A/B vs the generic segment kernel
python -m pytest tests/test_gpu_count.py tests/test_gpu_boundaries.py tests/test_gpu_frontier.py -q -x > gpurun_out/pytest7.log 2>&1; echo PYTEST_EXIT=$? >> gpurun_out/pytest7.log
python bench.py --no-cpu-baseline --no-secondary --no-e2e > gpurun_out/bench7.log 2>&1
