mkdir -p gpurun_out
for co in 100 75 50 35 25; do
  for ro in "" "--reorder"; do
    MAPI_CSR_CARVEOUT=$co timeout 900 python bench.py --workload cfg5 --steps 3 --warmup 2 --no-cpu-baseline $ro > gpurun_out/b5.log 2>&1; tail -1 gpurun_out/b5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('carveout $co $ro', round(d['value']))"
  done
done
