mkdir -p gpurun_out
B="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/plain5.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_rank -c 40 --csv --log-file gpurun_out/launches_cfg5.csv $B > gpurun_out/ncu_launch5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rank_rows_mp -s 3 -c 1 -o gpurun_out/prof_cfg5_rows $B > gpurun_out/ncu_full5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rank_normalize -s 3 -c 1 -o gpurun_out/prof_cfg5_norm $B > gpurun_out/ncu_full5n.log 2>&1
echo done
