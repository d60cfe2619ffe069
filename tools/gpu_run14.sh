#!/bin/bash
# --set full capture of the final D2 cnt_kernel (pass loop unrolled by 2) + config-5 launch list
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:cnt_kernel<unsigned long, \(bool\)1, \(bool\)1, \(bool\)1, \(int\)0, \(bool\)1>' -s 1 -c 1 -o gpurun_out/r02g_cnt_c5_d2 \
    python tools/run_config.py --config 5 --mode count --digest --reps 2 > gpurun_out/ncu_full_r02g.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_r02g.csv python tools/c5_once.py 5 > gpurun_out/ncu_launch_g.log 2>&1
ls -la gpurun_out | tail -4
