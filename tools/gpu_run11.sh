# evidence run of the round-2 build: full GPU suite, smoke, bench (default line), config-3 launch list + dfs_kernel capture
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r02.log 2>&1; echo PYTEST_EXIT=$? >> gpurun_out/pytest_gpu_r02.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02.log 2>&1; echo SMOKE_EXIT=$? >> gpurun_out/smoke_r02.log
python bench.py > gpurun_out/bench_r02.log 2>&1; echo BENCH_EXIT=$? >> gpurun_out/bench_r02.log
ncu --set full --clock-control none --import-source on -k regex:"dfs_kernel" -c 1 -o gpurun_out/r02_mat_c3_lp python tools/run_config.py --config 3 --reps 1 > gpurun_out/ncu_full11.log 2>&1
ls -la gpurun_out | tail -5
