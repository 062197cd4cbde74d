# K3s: plan-time bank-conflict-aware word order, A/B on cfg5 + parity tests of the planned path
mkdir -p gpurun_out
: > gpurun_out/r02_probe_k3s_deconflict.log
for dc in 0 1 2 3 5 8; do
  MAPI_PLAN_DECONFLICT=$dc timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dc_$dc.log 2>&1
  python - "$dc" <<'PY' >> gpurun_out/r02_probe_k3s_deconflict.log
import json,sys
dc=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/dc_{dc}.log").read().strip().splitlines()[-1])
    print(f"MAPI_PLAN_DECONFLICT={dc}: {d['value']:.1f} it/s ({1e3*d['ms_per_step']/200:.1f} us / iteration), plan build {d['plan_build']['repeat_s']*1e3:.1f} ms, tol 1e-7: {d['time_to_convergence']['iters']} iterations {d['time_to_convergence']['ms_median']:.3f} ms")
except Exception as e:
    print(dc, "ERR", e, open(f"gpurun_out/dc_{dc}.log").read()[-600:])
PY
done
cat gpurun_out/r02_probe_k3s_deconflict.log
timeout 1500 python -m pytest tests/test_gpu_rank_plan.py -x -q -m gpu > gpurun_out/pytest_plan_dc.log 2>&1; echo "pytest plan rc=$?"; tail -3 gpurun_out/pytest_plan_dc.log
# phase trace with and without
for dc in 0 3; do MAPI_PLAN_DECONFLICT=$dc MAPI_PLAN_TRACE=1 timeout 600 python bench.py --workload cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/dc_trace_$dc.log 2>&1; grep -i "phase\|trace" gpurun_out/dc_trace_$dc.log | head -5; done
# ncu: shared-memory wavefronts / conflicts of the planned kernel with the new order
C="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_rank_plan -c 2 --csv --log-file gpurun_out/r02_cfg5_k3s_deconflict_metrics.csv $C > gpurun_out/ncu_dc.log 2>&1; echo "ncu rc=$?"
tail -4 gpurun_out/r02_cfg5_k3s_deconflict_metrics.csv | cut -c1-400
