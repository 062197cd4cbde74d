mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rank_plan.py -x -q -m gpu > gpurun_out/pytest_plan_sb2.log 2>&1; echo "pytest plan rc=$?"; tail -2 gpurun_out/pytest_plan_sb2.log
for i in 1 2; do timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --cpu-seconds 8 > gpurun_out/r2_bench_cfg5_sb$i.log 2>&1; echo "cfg5 rc=$?"; done
timeout 600 python bench.py --workload cfg5 --op dot --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_dot_sb.log 2>&1; echo "cfg5 dot rc=$?"
MAPI_PLAN_SLOT_BLOCK=16384 timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_sb16k.log 2>&1; echo "cfg5 16k rc=$?"
python - <<'PY'
import json
for w in ["cfg5_sb1","cfg5_sb2","cfg5_dot_sb","cfg5_sb16k"]:
    d=json.loads(open(f"gpurun_out/r2_bench_{w}.log").read().strip().splitlines()[-1])
    open(f"gpurun_out/r02_bench_{w}.json","w").write(json.dumps(d)+"\n")
    print(w, round(d["value"],1), "us/it", round(1e3*d["ms_per_step"]/200,1), "frac", round(d["roofline"]["frac"],4), "ttc", d["time_to_convergence"]["ms_median"], d["time_to_convergence"]["iters"], "plan", round(d["plan_build"]["repeat_s"]*1e3,1), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
C="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rank_plan -c 1 -f -o gpurun_out/r02_cfg5_k3s $C > gpurun_out/ncu_full_cfg5.log 2>&1; echo "ncu rc=$?"
