mkdir -p gpurun_out
timeout 900 python -m pytest -q -x --timeout 600 tests/test_gpu_rank_plan.py -k "not cfg5" > gpurun_out/r2_plan3_tests.log 2>&1; tail -3 gpurun_out/r2_plan3_tests.log
MAPI_PLAN_TRACE=1 timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_plan3.json 2> gpurun_out/r2_bench_cfg5_plan3.err; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_cfg5_plan3.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d.get('time_to_convergence'))"; grep "plan trace" gpurun_out/r2_bench_cfg5_plan3.err | tail -3
