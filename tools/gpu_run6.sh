# D2 kernel at CNT_D2_POPS=2: count parity, full bench line, config-5 launch list and --set full capture of the D2 kernel
python -m pytest tests/test_gpu_count.py tests/test_gpu_boundaries.py -q -x > gpurun_out/pytest_count6.log 2>&1; echo PYTEST_EXIT=$? >> gpurun_out/pytest_count6.log
python bench.py > gpurun_out/bench6.log 2>&1; echo EXIT=$? >> gpurun_out/bench6.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_d2.csv python tools/c5_once.py 5 > gpurun_out/ncu_launch6.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:cnt_kernel<unsigned long, \(bool\)1, \(bool\)1, \(bool\)1, \(int\)0, \(bool\)1>' -s 1 -c 1 -o gpurun_out/r02_cnt_c5d2 \
    python tools/run_config.py --config 5 --mode count --digest --reps 2 > gpurun_out/ncu_full6.log 2>&1
ls -la gpurun_out/
