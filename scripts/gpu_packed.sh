mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x -k "host_many" --timeout 600 > gpurun_out/pytest_packed.log 2>&1; tail -3 gpurun_out/pytest_packed.log
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/bench_default.log 2>&1; echo "rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_default.log").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], d["e2e"]["h2d_bytes_per_step"], "clk", d["clocks"])
PY
