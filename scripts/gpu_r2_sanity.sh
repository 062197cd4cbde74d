# last sanity pass on the final build: ranking tests (plan, sharded, CSR), smoke, cfg5 and default bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_rank_plan.py tests/test_gpu_rank_sharded.py tests/test_gpu_rank.py -x -q -m gpu > gpurun_out/pytest_rank_final.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_rank_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --cpu-seconds 8 > gpurun_out/r2_bench_cfg5.log 2>&1; echo "cfg5 rc=$?"
timeout 900 python bench.py > gpurun_out/r2_bench_default.log 2>&1; echo "default rc=$?"
python - <<'PY'
import json
for w in ["cfg5","default"]:
    d=json.loads(open(f"gpurun_out/r2_bench_{w}.log").read().strip().splitlines()[-1])
    open(f"gpurun_out/r02_bench_{w}_final.json","w").write(json.dumps(d)+"\n")
    print(w, round(d["value"],1), "frac", round(d["roofline"]["frac"],4), "traffic", d["roofline"].get("traffic"), "e2e", (d.get("e2e") or {}).get("value"), d["clocks"])
PY
