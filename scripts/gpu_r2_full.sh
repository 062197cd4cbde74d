# round 2: full GPU suite + smoke + every workload's bench line
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/r2_pytest_all.log 2>&1; tail -3 gpurun_out/r2_pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r2_bench_default.log 2>&1; echo "default rc=$?"
for w in cfg1 cfg2 cfg4 cfg5 mincov mincov_k4096 alg2; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --cpu-seconds 8 > gpurun_out/r2_bench_$w.log 2>&1; echo "$w rc=$?"
done
timeout 600 python bench.py --workload cfg5 --op dot --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_dot.log 2>&1; echo "cfg5 dot rc=$?"
for md in sym_p2p p2p sharded; do
  timeout 600 python bench.py --mode $md --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_$md.log 2>&1; echo "$md rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference.log 2>&1; echo "ref rc=$?"
python - <<'PY'
import json
for w in ["default","cfg1","cfg2","cfg4","cfg5","cfg5_dot","mincov","mincov_k4096","alg2","sym_p2p","p2p","sharded","reference"]:
    try:
        d=json.loads(open(f"gpurun_out/r2_bench_{w}.log").read().strip().splitlines()[-1])
        r=d.get("roofline",{})
        print(w, round(d["value"],2), d["unit"], "frac", round(r.get("frac",0) or 0,3), r.get("unit"), "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"), "clk", (d.get("clocks") or {}).get("sm_mhz"))
        open(f"gpurun_out/r02_bench_{w}.json","w").write(json.dumps(d)+"\n")
    except Exception as e:
        print(w, "ERR", e)
PY
