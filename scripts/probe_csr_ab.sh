# A/B of the current libmapi against scripts/bin/libmapi_prev.so on cfg5 (+ rank tests on current)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rank.py -q -x > gpurun_out/pytest_rank.log 2>&1; tail -1 gpurun_out/pytest_rank.log
cp paper_2110_12065_b200/libmapi.so /tmp/libmapi_cur.so
for v in cur prev cur2; do
  if [ "$v" = prev ]; then cp scripts/bin/libmapi_prev.so paper_2110_12065_b200/libmapi.so; else cp /tmp/libmapi_cur.so paper_2110_12065_b200/libmapi.so; fi
  timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_$v.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/bench_cfg5_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), d['ms_per_step'], d['roofline'].get('kernel_ms_avg'))"
done
