mkdir -p gpurun_out
timeout 600 python bench.py --workload alg3 --steps 20 --warmup 3 > gpurun_out/r02_bench_alg3.json 2> gpurun_out/r02_bench_alg3.err; tail -2 gpurun_out/r02_bench_alg3.err; tail -c 1500 gpurun_out/r02_bench_alg3.json
timeout 600 python bench.py --workload alg3 --op dot --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_alg3_dot.json 2>/dev/null
timeout 900 python bench.py > gpurun_out/r02_bench_default_b.json 2> gpurun_out/r02_bench_default_b.err; tail -2 gpurun_out/r02_bench_default_b.err; python -c "
import json; d=json.loads(open('gpurun_out/r02_bench_default_b.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline'].get('frac_of_read_ceiling_7200'), d['full_matrix_path'], d['e2e']['value'])"
