"""Per-iteration cost of the pieces of the row-sharded MAPI step at N = 1 (investigation)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_12065_b200 as m
import synth
m.load()
n = 32768
A = synth.cfg3(device="cuda")["A"]
w = torch.full((n,), 1 / np.sqrt(n), device="cuda")
y = torch.empty(n, device="cuda"); yf = torch.empty(n, device="cuda")
s = torch.empty(1, device="cuda"); d = torch.empty(1, device="cuda"); st = torch.empty(1, dtype=torch.int32, device="cuda")
def t(fn, reps=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
print(f"matvec (K1, 32768 rows): {t(lambda: m.mavp_matvec(A, w, y)):8.1f} us")
print(f"normalize (1 CTA):       {t(lambda: m.normalize(y, w.clone(), s, d, st)):8.1f} us")
print(f"copy y (world-1 gather): {t(lambda: yf.copy_(y)):8.1f} us")
r = m.iterate(A, w, 1)
m.set_profiling(True); m.iterate(A, w, 10); print(f"coop iterate per iteration: {m.last_kernel_ms()*100:8.1f} us")
