mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -q -x -k "sym" --timeout 600 > gpurun_out/pytest_sym.log 2>&1; tail -3 gpurun_out/pytest_sym.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DMAPI_SYM_TRACE -o /tmp/p scripts/probe_k2s.cu && timeout 120 /tmp/p | tee gpurun_out/probe_k2s.log
timeout 300 python - <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2110_12065_b200 as m, synth
m.load()
cfg = synth.cfg3(device="cuda")
A = cfg["A"]; b0 = torch.from_numpy(cfg["b0"]).cuda()
for name, fn in [("full", m.iterate), ("sym", m.iterate_sym)]:
    fn(A, b0, 100); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): fn(A, b0, 100)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name}: {ms:.2f} ms / 100 iterations = {100 / (ms / 1e3):.0f} it/s", flush=True)
PY
