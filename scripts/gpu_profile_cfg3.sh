mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -k cfg3 > gpurun_out/pytest_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cfg3.log
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv $B > gpurun_out/ncu_launch.log 2>&1
$B > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_iterate_persistent -c 1 -o gpurun_out/prof_cfg3 $B > gpurun_out/ncu_full.log 2>&1
echo done
