# A/B: LEAN materializing DFS step as one predicated stream (LEAN_PRED=1) vs branches; config 3 materialized
for v in "" lp "" lp; do
  TPGEN_LIB_VARIANT=$v python bench.py --workload config3 --no-cpu-baseline --no-e2e --steps 10 >> gpurun_out/bench10_${v:-base}.log 2>&1
done
TPGEN_LIB_VARIANT=lp python -m pytest tests/test_gpu_parity.py tests/test_gpu_count.py -q -x -k "not config5" > gpurun_out/pytest10_lp.log 2>&1; echo EXIT=$? >> gpurun_out/pytest10_lp.log
