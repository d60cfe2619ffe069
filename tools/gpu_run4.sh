# A/B of the D2 pass structure: CNT_D2_POPS = 0 (default lib) / 1 / 2 -- config-5 bench (digest printed) + count parity corpus
for v in "" p1 p2; do
  TPGEN_LIB_VARIANT=$v python bench.py --no-cpu-baseline --no-secondary --no-e2e > gpurun_out/bench4_${v:-p0}.log 2>&1
  TPGEN_LIB_VARIANT=$v python -m pytest tests/test_gpu_count.py -q -x -k "matches_oracle or per_start or overflow" > gpurun_out/pytest4_${v:-p0}.log 2>&1
done
