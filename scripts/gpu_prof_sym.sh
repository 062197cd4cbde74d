mkdir -p gpurun_out
cat > /tmp/sym_once.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2110_12065_b200 as m, synth
m.load()
cfg = synth.cfg3(device="cuda")
A = cfg["A"]; b0 = torch.from_numpy(cfg["b0"]).cuda()
m.iterate_sym(A, b0, 10)
torch.cuda.synchronize()
PY
python /tmp/sym_once.py && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iterate_sym -c 1 -o gpurun_out/prof_cfg3_sym python /tmp/sym_once.py > gpurun_out/ncu_sym.log 2>&1; echo "ncu rc=$?"
