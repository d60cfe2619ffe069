python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_EXIT=$? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo SMOKE_EXIT=$? >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; echo BENCH_EXIT=$? >> gpurun_out/bench.log
