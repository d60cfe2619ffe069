# D2 count kernel: count-mode parity (incl. config 5 every start vertex) and the config-5 bench, A/B vs TPGEN_NO_D2
python -m pytest tests/test_gpu_count.py tests/test_gpu_boundaries.py -q -x > gpurun_out/pytest_count.log 2>&1; echo PYTEST_EXIT=$? >> gpurun_out/pytest_count.log
python bench.py --no-cpu-baseline --no-secondary > gpurun_out/bench_d2.log 2>&1; echo EXIT=$? >> gpurun_out/bench_d2.log
TPGEN_NO_D2=1 python bench.py --no-cpu-baseline --no-secondary > gpurun_out/bench_nod2.log 2>&1; echo EXIT=$? >> gpurun_out/bench_nod2.log
