mkdir -p gpurun_out
for cfgname in "persist0-orig:MAPI_CSR_HUB=2" "nohub-orig:MAPI_CSR_HUB=0"; do
  name=${cfgname%%:*}; envv=${cfgname#*:}
  env $envv timeout 900 python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-reorder > gpurun_out/bench_cfg5_$name.log 2>&1; tail -1 gpurun_out/bench_cfg5_$name.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', d['value'])"
done
B="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline --no-reorder"
timeout 900 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.sum,smsp__inst_executed.sum --clock-control none -k regex:k_rank_rows -c 4 $B 2>&1 | grep -E "k_rank_rows|duration|warps_active|wavefronts|inst_executed" | head -24
