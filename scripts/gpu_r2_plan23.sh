mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x --timeout 600 tests/test_gpu_rank_plan.py 2>&1 | tail -3
for i in 1 2; do
MAPI_PLAN_TRACE=1 timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2> gpurun_out/r2_plan23.err > gpurun_out/r2_plan23.json; grep "plan trace" gpurun_out/r2_plan23.err | tail -1; python -c "
import json; d=json.loads(open('gpurun_out/r2_plan23.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d.get('time_to_convergence',{}).get('ms_median'))"
done
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('untraced', d['value'], d['roofline']['frac'], d.get('time_to_convergence',{}).get('ms_median'))"
