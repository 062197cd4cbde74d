mkdir -p gpurun_out
CMD="python bench.py --workload cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
(cd _old && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rank_plan -c 1 -f -o $GRAFT_REPO_ROOT/gpurun_out/ncu_plan_old $CMD > $GRAFT_REPO_ROOT/gpurun_out/ncu_plan_old.log 2>&1)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rank_plan -c 1 -f -o gpurun_out/ncu_plan_new $CMD > gpurun_out/ncu_plan_new.log 2>&1
ls -la gpurun_out/*.ncu-rep
