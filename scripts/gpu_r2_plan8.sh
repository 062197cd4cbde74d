mkdir -p gpurun_out
MAPI_PLAN_TRACE=1 timeout 600 python bench.py --workload cfg5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_cfg5_plan8.json 2> gpurun_out/r2_bench_cfg5_plan8.err; grep "plan trace" gpurun_out/r2_bench_cfg5_plan8.err | tail -2
