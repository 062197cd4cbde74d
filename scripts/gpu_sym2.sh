mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x -k "sym or host" --timeout 600 > gpurun_out/pytest_sym.log 2>&1; tail -3 gpurun_out/pytest_sym.log
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/bench_default.log 2>&1; echo "rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_default.log").read().strip().splitlines()[-1])
print("value", d["value"], "hbm", d["hbm_gbs"], "frac", d["roofline"]["frac"], "share", d["roofline"]["kernel_share_of_step"])
print("full", d["full_matrix_path"])
print("e2e", d["e2e"]["value"], d["e2e"]["ms_per_step"], "clk", d["clocks"], "cpu", d["cpu_baseline"]["value"])
PY
