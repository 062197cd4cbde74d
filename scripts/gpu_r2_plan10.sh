mkdir -p gpurun_out
timeout 900 python -m pytest -q -x --timeout 600 tests/test_gpu_rank_plan.py -k "not cfg5" 2>&1 | tail -2
MAPI_PLAN_TRACE=1 timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2> gpurun_out/r2_plan10.err > gpurun_out/r2_plan10.json; grep "plan trace" gpurun_out/r2_plan10.err | tail -2; python -c "
import json; d=json.loads(open('gpurun_out/r2_plan10.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d.get('time_to_convergence',{}).get('ms_median'))"
