mkdir -p gpurun_out
CMD="python bench.py --workload cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_plan.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rank_plan -c 1 -o gpurun_out/r2_plan_full2 $CMD > gpurun_out/ncu_plan_full2.log 2>&1; tail -3 gpurun_out/ncu_plan_full.log; ls -la gpurun_out/*.ncu-rep
