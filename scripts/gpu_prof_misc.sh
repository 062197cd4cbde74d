mkdir -p gpurun_out
B1="python bench.py --workload cfg1 --steps 1 --warmup 1 --no-cpu-baseline"
$B1 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_iterate_single -c 1 -o gpurun_out/prof_cfg1_k6t $B1 > /dev/null 2>&1; echo k6t $?
B2="python bench.py --workload cfg2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv $B2 > /dev/null 2>&1; echo cfg2 launches $?
