mkdir -p gpurun_out
B="python bench.py --workload cfg2 --steps 1 --warmup 1 --no-cpu-baseline"
$B > gpurun_out/plain2c.log 2>&1 && ncu --set full --clock-control none -k regex:k_iterate_persistent -s 2 -c 1 -o gpurun_out/prof_cfg2 $B > gpurun_out/ncu_cfg2.log 2>&1
echo done
