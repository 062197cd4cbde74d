mkdir -p gpurun_out
MAPI_PLAN_TRACE=1 MAPI_PLAN_TRACE_FILE=gpurun_out/r2_plan_cta.csv timeout 600 python bench.py --workload cfg5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_cfg5_plan4.json 2> gpurun_out/r2_bench_cfg5_plan4.err; grep "plan trace" gpurun_out/r2_bench_cfg5_plan4.err | tail -1; head -3 gpurun_out/r2_plan_cta.csv
