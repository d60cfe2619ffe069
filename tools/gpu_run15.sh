#!/bin/bash
# final HEAD check: full GPU suite, smoke, bench
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02h.log 2>&1; echo PYTEST_EXIT=$? >> gpurun_out/pytest_gpu_r02h.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02h.log 2>&1; echo SMOKE_EXIT=$? >> gpurun_out/smoke_r02h.log
python bench.py > gpurun_out/bench_r02h.json 2> gpurun_out/bench_r02h.err; echo BENCH_EXIT=$? >> gpurun_out/bench_r02h.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02h.json 2> gpurun_out/bench_ref_r02h.err
