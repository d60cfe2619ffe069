#!/bin/bash
# final evidence of the round-2 build (pass loop unrolled by 2): count-mode A/B on configs 3 and 5 (unroll 1 vs 2),
# full GPU suite, smoke, bench
bash tools/ab_count.sh unr1 base > gpurun_out/ab_count_unr.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02g.log 2>&1; echo PYTEST_EXIT=$? >> gpurun_out/pytest_gpu_r02g.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02g.log 2>&1; echo SMOKE_EXIT=$? >> gpurun_out/smoke_r02g.log
python bench.py > gpurun_out/bench_r02g.json 2> gpurun_out/bench_r02g.err; echo BENCH_EXIT=$? >> gpurun_out/bench_r02g.err
ls -la gpurun_out | tail -6
