# K3s word order: (lane chunk, fragment) groups (mode 1) vs whole fragments (mode 2), same box
mkdir -p gpurun_out
: > gpurun_out/r02_probe_k3s_deconflict2.log
for cfg in "0 1" "2 1" "1 2" "2 1" "1 2"; do
  set -- $cfg
  MAPI_PLAN_DECONFLICT=$1 MAPI_PLAN_DECONFLICT_MODE=$2 timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dc2.log 2>&1
  python - "$1" "$2" <<'PY' >> gpurun_out/r02_probe_k3s_deconflict2.log
import json,sys
try:
    d=json.loads(open("gpurun_out/dc2.log").read().strip().splitlines()[-1])
    print(f"passes {sys.argv[1]} mode {sys.argv[2]}: {d['value']:.1f} it/s ({1e3*d['ms_per_step']/200:.1f} us / iteration), plan build {d['plan_build']['repeat_s']*1e3:.1f} ms")
except Exception as e:
    print(sys.argv[1:], "ERR", e, open("gpurun_out/dc2.log").read()[-800:])
PY
done
cat gpurun_out/r02_probe_k3s_deconflict2.log
MAPI_PLAN_DECONFLICT_MODE=2 timeout 1500 python -m pytest tests/test_gpu_rank_plan.py -x -q -m gpu > gpurun_out/pytest_plan_dc2.log 2>&1; echo "pytest plan (mode 2) rc=$?"; tail -3 gpurun_out/pytest_plan_dc2.log
C="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
MAPI_PLAN_DECONFLICT_MODE=2 timeout 900 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum --clock-control none -k regex:k_rank_plan -c 2 --csv --log-file gpurun_out/r02_cfg5_k3s_deconflict2_metrics.csv $C > gpurun_out/ncu_dc2.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r02_cfg5_k3s_deconflict2_metrics.csv | cut -c150-400
