mkdir -p gpurun_out
B="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/plain5c.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_rank_rows_mp -s 3 -c 1 -o gpurun_out/prof_cfg5_rows3 $B > gpurun_out/ncu_rows3.log 2>&1
echo done
