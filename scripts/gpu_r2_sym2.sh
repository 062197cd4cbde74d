mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x --timeout 1200 tests/test_gpu_dense.py tests/test_gpu_sharded.py -k "sym or cfg3 or host_many" 2>&1 | tail -3
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DMAPI_SYM_TRACE -I include -o /tmp/p scripts/probe_k2s.cu && timeout 120 /tmp/p | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_sym_bench2.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2_sym_bench2.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['ms_per_step'], d.get('clocks'))"
