#!/bin/bash
# Round-2 ncu evidence (run under gpurun; part 1 or 2 -- gpurun_out must stay under 64 MiB):
# launch list of one config-5 COUNT_HASH call, --set full captures of the dominant kernels.
set -x
if [ "$1" = 1 ]; then
python tools/c5_once.py 5 > gpurun_out/p_c5.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c5.csv \
      python tools/c5_once.py 5 > gpurun_out/ncu_a.log 2>&1
python tools/run_config.py --config 5 --mode count --digest --reps 1 > gpurun_out/p5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:cnt_kernel -s 1 -c 1 -o gpurun_out/r02_cnt_c5 \
      python tools/run_config.py --config 5 --mode count --digest --reps 1 > gpurun_out/ncu_b.log 2>&1
python tools/run_config.py --config 3 --mode count --digest --reps 2 > gpurun_out/p3c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:cnt_kernel -s 1 -c 1 -o gpurun_out/r02_cnt_c3 \
      python tools/run_config.py --config 3 --mode count --digest --reps 2 > gpurun_out/ncu_c.log 2>&1
else
python tools/run_config.py --config 3 --reps 2 > gpurun_out/p3m.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"dfs_kernel|expand_fast" -s 2 -c 2 -o gpurun_out/r02_mat_c3 \
      python tools/run_config.py --config 3 --reps 2 > gpurun_out/ncu_d.log 2>&1
fi
ls -la gpurun_out/*.ncu-rep
