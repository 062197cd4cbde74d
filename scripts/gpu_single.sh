mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x -k "single or every_dense or cluster or smoke or cfg1" --timeout 600 > gpurun_out/pytest_single.log 2>&1; tail -3 gpurun_out/pytest_single.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python scripts/probe_small_range.py > gpurun_out/probe_small_range.log 2>&1; cat gpurun_out/probe_small_range.log
timeout 600 python bench.py --workload cfg1 --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_cfg1.log 2>&1; tail -1 gpurun_out/bench_cfg1.log | cut -c1-300
