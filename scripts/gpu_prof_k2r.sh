# K2r phase probe + ncu full capture of one K2r launch in the cfg2 bench step
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -DMAPI_RES_TRACE -o /tmp/p scripts/probe_k2r.cu && timeout 120 /tmp/p > gpurun_out/probe_k2r.log 2>&1; cat gpurun_out/probe_k2r.log
B="python bench.py --workload cfg2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_cfg2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate_resident -s 2 -c 1 -o gpurun_out/prof_cfg2_k2r $B > gpurun_out/ncu_full_k2r.log 2>&1; echo "ncu rc=$?"
