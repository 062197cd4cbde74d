# K2s in-stream L2 prefetch sweep (MAPI_SYM_STREAM_PF rows ahead), plan-build fix check
mkdir -p gpurun_out
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
: > gpurun_out/r02_probe_k2s_streampf.log
for pf in 0 8 16 24 32 48 0 16; do
  MAPI_SYM_STREAM_PF=$pf timeout 600 $B > gpurun_out/spf_$pf.log 2>&1
  python - "$pf" <<'PY' >> gpurun_out/r02_probe_k2s_streampf.log
import json,sys
pf=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/spf_{pf}.log").read().strip().splitlines()[-1])
    print(f"MAPI_SYM_STREAM_PF={pf:>3}: {d['value']:.1f} it/s, kernel {d['roofline']['kernel_ms_avg']:.3f} ms / 100 iterations, clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}, full-matrix K2c {d['full_matrix_path']['value']:.1f}")
except Exception as e:
    print(pf, "ERR", e)
PY
done
cat gpurun_out/r02_probe_k2s_streampf.log
MAPI_SYM_STREAM_PF=16 timeout 1200 python -m pytest tests/test_gpu_dense.py -x -q -m gpu -k "sym" > gpurun_out/pytest_sym_spf.log 2>&1; echo "pytest sym rc=$?"; tail -3 gpurun_out/pytest_sym_spf.log
timeout 1200 python -m pytest tests/test_gpu_rank_plan.py -x -q -m gpu > gpurun_out/pytest_plan.log 2>&1; echo "pytest plan rc=$?"; tail -3 gpurun_out/pytest_plan.log
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_b.log 2>&1; echo "cfg5 rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench_cfg5_b.log").read().strip().splitlines()[-1])
print("cfg5", d["value"], d["plan_build"], d["time_to_convergence"]["ms_median"])
PY
