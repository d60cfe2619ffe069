# A/B of CNT_D2_POPS = 2 / 3 / 4 on one box (config-5 bench, digest checked in the log)
for v in p2 p3 p4 p2; do
  TPGEN_LIB_VARIANT=$v python bench.py --no-cpu-baseline --no-secondary --no-e2e > gpurun_out/bench5_$v.log 2>&1
done
