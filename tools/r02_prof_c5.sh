#!/bin/bash
# --set full capture of the config-5 prime-path phase kernel (cnt_kernel<uint64,TS,HSH,HX,P_PP>).
python tools/run_config.py --config 5 --mode count --digest --reps 2 > gpurun_out/p5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k 'regex:cnt_kernel<unsigned long, \(bool\)1, \(bool\)1, \(bool\)1, \(int\)0>' -s 1 -c 1 -o gpurun_out/r02_cnt_c5pp \
      python tools/run_config.py --config 5 --mode count --digest --reps 2 > gpurun_out/ncu_e.log 2>&1
ls -la gpurun_out/*.ncu-rep; tail -3 gpurun_out/ncu_e.log
