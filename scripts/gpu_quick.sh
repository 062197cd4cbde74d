mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pca.py tests/test_gpu_dense.py -q -x -k "pca or resident" --timeout 600 > gpurun_out/pytest_quick.log 2>&1; tail -2 gpurun_out/pytest_quick.log
for w in cfg2; do
timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.log 2>&1; tail -1 gpurun_out/bench_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'])"
MAPI_PCA_FUSE=0 timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${w}_nofuse.log 2>&1; tail -1 gpurun_out/bench_${w}_nofuse.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w nofuse', d['value'], d['ms_per_step'])"
done
