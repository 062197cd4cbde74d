# round-end style refresh: full GPU suite, smoke, every bench line, ncu launch list + full capture of K2s
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_all.log 2>&1; tail -3 gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "default rc=$?"
for w in cfg1 cfg2 cfg4 cfg5 mincov mincov_k4096 alg2; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --cpu-seconds 8 > gpurun_out/bench_$w.log 2>&1; echo "$w rc=$?"
done
timeout 600 python bench.py --mode p2p --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p2p.log 2>&1; echo "p2p rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
python - <<'PY'
import json
for w in ["default","cfg1","cfg2","cfg4","cfg5","mincov","mincov_k4096","alg2","p2p","reference"]:
    try:
        d=json.loads(open(f"gpurun_out/bench_{w}.log").read().strip().splitlines()[-1])
        r=d.get("roofline",{})
        print(w, round(d["value"],2), d["unit"], "frac", round(r.get("frac",0),3), r.get("unit"), "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"), "clk", (d.get("clocks") or {}).get("sm_mhz"))
        open(f"gpurun_out/r01_bench_{w}.json","w").write(json.dumps(d)+"\n")
    except Exception as e:
        print(w, "ERR", e)
PY
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_iterate_sym -c 1 -o gpurun_out/prof_cfg3_sym100 $B > gpurun_out/ncu_full_sym.log 2>&1; echo "full rc=$?"
echo done
