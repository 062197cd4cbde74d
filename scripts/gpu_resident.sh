# K2r parity + cfg2 bench + n sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_pca.py -q -x --timeout 600 > gpurun_out/pytest_resident.log 2>&1; tail -3 gpurun_out/pytest_resident.log
timeout 600 python bench.py --workload cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_res.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/bench_cfg2_res.log | cut -c1-330
timeout 600 python scripts/probe_resident_range.py > gpurun_out/probe_resident_range.log 2>&1; cat gpurun_out/probe_resident_range.log
