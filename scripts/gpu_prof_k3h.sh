mkdir -p gpurun_out
B="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none -k regex:k_rank_rows_mp -s 3 -c 1 -o gpurun_out/prof_k3 $B > /dev/null 2>&1; echo k3 $?
MAPI_CSR_HUB=2 timeout 900 ncu --set full --clock-control none -k regex:k_rank_rows_mp -s 3 -c 1 -o gpurun_out/prof_k3h0 $B > /dev/null 2>&1; echo k3h0 $?
