mkdir -p gpurun_out
timeout 900 python -m pytest -q -x --timeout 600 tests/test_gpu_rank_plan.py > gpurun_out/r2_plan9_tests.log 2>&1; tail -15 gpurun_out/r2_plan9_tests.log
MAPI_PLAN_TRACE=1 MAPI_PLAN_TRACE_FILE=gpurun_out/r2_plan9_cta.csv timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_cfg5_plan5.json 2> gpurun_out/r2_bench_cfg5_plan5.err; grep "plan trace" gpurun_out/r2_bench_cfg5_plan5.err | tail -1
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_plan5b.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_cfg5_plan5b.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d.get('time_to_convergence'), d.get('plan_build'))"
MAPI_PLAN_TRACE=1 timeout 600 python bench.py --workload cfg5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 >/dev/null | grep "plan trace" | tail -2
