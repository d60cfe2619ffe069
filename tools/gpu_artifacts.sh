set -x
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_EXIT=$? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_c3.log 2>&1
python bench.py --engine frontier --no-cpu-baseline > gpurun_out/bench_fr.log 2>&1
python bench.py --count --no-cpu-baseline > gpurun_out/bench_cnt.log 2>&1
python bench.py --workload config5 > gpurun_out/bench_c5.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
python tools/bench_stages.py > gpurun_out/stages.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python tools/run_config.py --config 3 --reps 3 > gpurun_out/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_fr.csv python bench.py --engine frontier --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fr.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"dfs_kernel|expand_fast" -c 2 -o gpurun_out/prof_c3 python tools/run_config.py --config 3 --reps 1 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:frontier_level_kernel -s 16 -c 1 -o gpurun_out/prof_fr python bench.py --engine frontier --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fr_full.log 2>&1
ls -la gpurun_out
