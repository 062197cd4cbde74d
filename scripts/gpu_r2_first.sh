# round 2 re-entry: new parity tests, K3s plan tests, cfg5 plan bench, default bench
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest -q -x --timeout 600 tests/test_gpu_rank_plan.py > gpurun_out/r2_plan_tests.log 2>&1; tail -3 gpurun_out/r2_plan_tests.log
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_plan.json 2> gpurun_out/r2_bench_cfg5_plan.err; tail -c 2500 gpurun_out/r2_bench_cfg5_plan.json; tail -3 gpurun_out/r2_bench_cfg5_plan.err
timeout 600 python bench.py --workload cfg5 --csr-path k3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_k3.json 2>&1; tail -c 600 gpurun_out/r2_bench_cfg5_k3.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:k_rank_plan -c 1 --csv python bench.py --workload cfg5 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_plan.csv 2>&1; tail -20 gpurun_out/r2_ncu_plan.csv
timeout 2400 python -m pytest -q --timeout 1200 -m gpu tests/test_gpu_dense.py tests/test_gpu_batched.py tests/test_gpu_rank.py tests/test_gpu_pca.py -k "cfg3_end_to_end or cfg4_full or fixed_200 or nonfinite or cfg2" > gpurun_out/r2_parity.log 2>&1; tail -5 gpurun_out/r2_parity.log
