mkdir -p gpurun_out
for pf in 0 16 24 32 48 64 0 32; do
MAPI_SYM_PREFETCH=$pf timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('prefetch_rows $pf:', round(d['value'],1), 'it/s', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done | tee gpurun_out/r02_probe_k2s_prefetch.log
MAPI_SYM_PREFETCH=32 timeout 900 python -m pytest -q -x --timeout 600 tests/test_gpu_dense.py -k "sym" 2>&1 | tail -3
