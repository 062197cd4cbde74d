mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_pca.py tests/test_gpu_random.py -q -x -k "resident or pca or random" --timeout 600 > gpurun_out/pytest_quick.log 2>&1; tail -1 gpurun_out/pytest_quick.log
for i in 1 2; do
timeout 600 python bench.py --workload cfg2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1; tail -1 gpurun_out/bench_cfg2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', round(d['value']), d['ms_per_step'])"
done
