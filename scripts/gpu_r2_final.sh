# round 2 final refresh: every workload's bench line, the reference arm, ncu launch lists and full captures
mkdir -p gpurun_out
for w in cfg1 cfg2 cfg4 cfg5 mincov mincov_k4096 alg2 alg3; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --cpu-seconds 8 > gpurun_out/r2_bench_$w.log 2>&1; echo "$w rc=$?"
done
timeout 600 python bench.py --workload cfg5 --op dot --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_dot.log 2>&1; echo "cfg5 dot rc=$?"
for md in sym_p2p p2p sharded; do
  timeout 600 python bench.py --mode $md --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_$md.log 2>&1; echo "$md rc=$?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_reference.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/r2_bench_default.log 2>&1; echo "default rc=$?"
python - <<'PY'
import json
for w in ["default","cfg1","cfg2","cfg4","cfg5","cfg5_dot","mincov","mincov_k4096","alg2","alg3","sym_p2p","p2p","sharded","reference"]:
    try:
        d=json.loads(open(f"gpurun_out/r2_bench_{w}.log").read().strip().splitlines()[-1])
        r=d.get("roofline") or {}
        print(w, round(d["value"],2), d["unit"], "frac", round(r.get("frac",0) or 0,4), r.get("unit"), "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"), "clk", (d.get("clocks") or {}).get("sm_mhz"), (d.get("clocks") or {}).get("reasons"))
        open(f"gpurun_out/r02_bench_{w}.json","w").write(json.dumps(d)+"\n")
    except Exception as e:
        print(w, "ERR", e)
PY
# ncu: launch lists of the default bench command and of cfg5, then one full capture each of K2s and K3s
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain_cfg3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg3.csv $B > gpurun_out/ncu_launch_cfg3.log 2>&1
$B > gpurun_out/plain_cfg3b.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate_sym -c 1 -f -o gpurun_out/r02_cfg3_sym $B > gpurun_out/ncu_full_cfg3.log 2>&1
C="python bench.py --workload cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$C > gpurun_out/plain_cfg5.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg5.csv $C > gpurun_out/ncu_launch_cfg5.log 2>&1
$C > gpurun_out/plain_cfg5b.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rank_plan -c 1 -f -o gpurun_out/r02_cfg5_k3s $C > gpurun_out/ncu_full_cfg5.log 2>&1
D="python bench.py --workload alg3 --steps 2 --warmup 1 --no-cpu-baseline"
$D > gpurun_out/plain_alg3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_alg3.csv $D > gpurun_out/ncu_launch_alg3.log 2>&1
ls -la gpurun_out/*.ncu-rep
echo done
