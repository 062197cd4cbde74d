"""Alg. 2 end to end on the synthetic occluded images under the two readings of steps 6/8
(l1-unit vs l2-unit MAPI outputs) and for min1 / min2 / dot (investigation; R11)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2110_12065_b200 as m
import synth

def psnr(a, b):
    return 10 * np.log10(1.0 / np.mean((a - b) ** 2))

m.load()
V_raw, img = synth.occluded_copies()
Vd = torch.from_numpy(V_raw).cuda()
clean = img.reshape(-1)
p_occ = np.mean([psnr(clean, V_raw[:, i]) for i in range(10)])
print(f"occluded copies: {p_occ:.2f} dB   mean image: {psnr(clean, V_raw.mean(axis=1)):.2f} dB")
def main():
  for opname, op in (("min1", 0), ("min2", 1), ("dot", 2)):
    for norm in ("l1", "l2"):
        try:
            run(opname, op, norm)
        except Exception as e:  # noqa: BLE001
            print(f"{opname:5s} {norm}: failed: {e}")

def run(opname, op, norm):
    if True:
        torch.cuda.synchronize(); t0 = time.perf_counter()
        Vc, mean = m.center_rows(Vd)
        C = m.min_covariance(Vc, op=0 if op == 2 else op) if op != 2 else (Vc @ Vc.T) / 9.0
        b0 = torch.full((16384,), 1.0 / 128.0, device="cuda")
        r1 = m.iterate(C, b0, 100, op=op)
        w1 = r1.w_l2 if (norm == "l2" or op == 2) else r1.w
        D = m.mavp_deflate(C, w1, op=op)
        r2 = m.iterate(D, b0, 100, op=op)
        w2 = r2.w_l2 if (norm == "l2" or op == 2) else r2.w
        W = torch.stack([w1, w2], 1).contiguous()
        Vh, _ = m.mavp_reconstruct(W, Vd, op=op)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        Vh = np.clip(Vh.cpu().numpy(), 0, 1)
        p = np.mean([psnr(clean, Vh[:, i]) for i in range(10)])
        print(f"{opname:5s} {norm}: reconstruction {p:6.2f} dB   pipeline {dt*1e3:7.1f} ms")

main()
