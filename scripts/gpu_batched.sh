mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batched.py -m gpu -q --timeout 600 -x > gpurun_out/pytest_batched.log 2>&1; tail -3 gpurun_out/pytest_batched.log
B="python bench.py --workload cfg4 --steps 3 --warmup 2 --no-cpu-baseline"
$B > gpurun_out/bench_cfg4b.log 2>&1; tail -1 gpurun_out/bench_cfg4b.log | cut -c1-1200
B1="python bench.py --workload cfg4 --steps 1 --warmup 1 --no-cpu-baseline"
$B1 > gpurun_out/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_batched_streamk -s 5 -c 1 -o gpurun_out/prof_cfg4_streamk $B1 > gpurun_out/ncu_full4.log 2>&1
B5="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline"
$B5 > gpurun_out/plain5b.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_rank -c 40 --csv --log-file gpurun_out/launches_cfg5b.csv $B5 > gpurun_out/ncu_launch5b.log 2>&1
echo done
