#!/bin/bash
# evidence run of the final round-2 build: full GPU suite, smoke, bench, config-5 launch list, --set full of the D2 cnt_kernel
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02f.log 2>&1; echo PYTEST_EXIT=$? >> gpurun_out/pytest_gpu_r02f.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02f.log 2>&1; echo SMOKE_EXIT=$? >> gpurun_out/smoke_r02f.log
python bench.py > gpurun_out/bench_r02f.json 2> gpurun_out/bench_r02f.err; echo BENCH_EXIT=$? >> gpurun_out/bench_r02f.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_r02f.csv python tools/c5_once.py 5 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:cnt_kernel<unsigned long, \(bool\)1, \(bool\)1, \(bool\)1, \(int\)0, \(bool\)1>' -s 1 -c 1 -o gpurun_out/r02f_cnt_c5_d2 \
    python tools/run_config.py --config 5 --mode count --digest --reps 2 > gpurun_out/ncu_full_r02f.log 2>&1
ls -la gpurun_out | tail -8
