# K2r (on-chip resident matrix) parity + cfg2 bench + ncu launch list of the cfg2 step
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_pca.py -q -x --timeout 600 > gpurun_out/pytest_resident.log 2>&1; tail -3 gpurun_out/pytest_resident.log
timeout 600 python bench.py --workload cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_res.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/bench_cfg2_res.log | cut -c1-300
B="python bench.py --workload cfg2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/ncu_launch_cfg2.log 2>&1; echo "ncu rc=$?"
