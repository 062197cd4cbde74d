# round 2, last refresh: the whole GPU suite + smoke, then every bench line / launch list / capture of gpu_r2_final.sh,
# then the sharded cfg5 line (world 1)
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_all.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
bash scripts/gpu_r2_final.sh
timeout 900 python bench.py --workload cfg5 --csr-path shard --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_bench_cfg5_shard.log 2>&1; echo "cfg5 shard rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench_cfg5_shard.log").read().strip().splitlines()[-1])
open("gpurun_out/r02_bench_cfg5_shard_world1.json","w").write(json.dumps(d)+"\n")
print("cfg5 shard", d["value"], d["roofline"]["frac"])
PY
