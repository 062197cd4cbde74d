mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_rank.py -q -x --timeout 900 > gpurun_out/pytest_rank.log 2>&1; tail -2 gpurun_out/pytest_rank.log
timeout 900 python bench.py --workload cfg5 --steps 5 --warmup 3 --cpu-seconds 8 > gpurun_out/bench_cfg5.log 2>&1; tail -1 gpurun_out/bench_cfg5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg5', d['value'], d['roofline']['frac'])"
