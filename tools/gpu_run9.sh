# A/B: D2 pops with predicates folded into multiplier / shift (CNT_D2_SELFREE=1) vs selects
for v in "" sf "" sf; do
  TPGEN_LIB_VARIANT=$v python bench.py --no-cpu-baseline --no-secondary --no-e2e --steps 5 >> gpurun_out/bench9_${v:-base}.log 2>&1
done
TPGEN_LIB_VARIANT=sf python -m pytest tests/test_gpu_count.py -q -x -k "matches_oracle or per_start or overflow" > gpurun_out/pytest9_sf.log 2>&1
