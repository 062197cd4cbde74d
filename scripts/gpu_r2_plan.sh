mkdir -p gpurun_out
timeout 900 python -m pytest -q -x --timeout 600 tests/test_gpu_rank_plan.py -k "not cfg5" > gpurun_out/r2_plan_tests.log 2>&1; tail -3 gpurun_out/r2_plan_tests.log
timeout 300 python -m pytest -q --timeout 300 tests/test_gpu_dense.py -k nonfinite > gpurun_out/r2_nonfinite.log 2>&1; tail -1 gpurun_out/r2_nonfinite.log
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_plan.json 2> gpurun_out/r2_bench_cfg5_plan.err; tail -c 1500 gpurun_out/r2_bench_cfg5_plan.json; tail -3 gpurun_out/r2_bench_cfg5_plan.err
timeout 900 python -m pytest -q --timeout 900 tests/test_gpu_rank_plan.py -k "cfg5" > gpurun_out/r2_plan_cfg5.log 2>&1; tail -3 gpurun_out/r2_plan_cfg5.log
PYTHONPATH=. timeout 900 python scripts/probe_cfg2_norms.py > gpurun_out/r2_cfg2_norms.log 2>&1; tail -12 gpurun_out/r2_cfg2_norms.log
