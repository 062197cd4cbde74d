mkdir -p gpurun_out
timeout 1200 python -m pytest -q -x --timeout 900 tests/test_gpu_dense.py -k "host_many" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_e2e.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_e2e.json').read().strip().splitlines()[-1]); e=d['e2e']; print(d['value'], 'e2e', e['value'], e['ms_per_step'], 'packed', e['packed']['value'], e['packed']['host_pack_s_once'])"
timeout 900 python bench.py --workload cfg5 --op dot --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_dot.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_cfg5_dot.json').read().strip().splitlines()[-1]); print('cfg5 dot', d['value'], d.get('time_to_convergence'), d.get('energy'))"
