mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b5.log 2>&1; tail -1 gpurun_out/b5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5 L1KEEP', round(d['value']))"
done
