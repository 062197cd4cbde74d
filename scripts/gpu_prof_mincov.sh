mkdir -p gpurun_out
B="python bench.py --workload mincov --steps 1 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/plain_mc.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_mavp_matmat -s 1 -c 1 -o gpurun_out/prof_mincov $B > gpurun_out/ncu_mc.log 2>&1
echo done
