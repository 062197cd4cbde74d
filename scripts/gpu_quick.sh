mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_pca.py -q -x --timeout 600 > gpurun_out/pytest_quick.log 2>&1; tail -2 gpurun_out/pytest_quick.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --workload cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg1.log 2>&1; tail -1 gpurun_out/bench_cfg1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', d['value'], d['ms_per_step'], d['roofline']['kernel_share_of_step'], d['gpu_launches'])"
