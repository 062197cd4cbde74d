mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_pca.py -q -x --timeout 600 > gpurun_out/pytest_quick.log 2>&1; tail -1 gpurun_out/pytest_quick.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for w in cfg1 cfg2; do
timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; tail -1 gpurun_out/bench_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']), d['ms_per_step'], d['roofline']['kernel_share_of_step'])"
done
