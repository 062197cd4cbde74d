mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dense.py tests/test_gpu_pca.py -m gpu -q --timeout 600 > gpurun_out/pytest_dense_rpi.log 2>&1; tail -2 gpurun_out/pytest_dense_rpi.log
for op in min1 dot min2 min1; do
  timeout 600 python bench.py --op $op --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_op_$op.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/bench_op_$op.log').read().strip().splitlines()[-1])
print('$op', round(d['value'],1), round(d['hbm_gbs'],1), d.get('energy'), d['clocks'])"
done
