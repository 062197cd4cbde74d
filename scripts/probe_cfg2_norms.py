"""cfg2 (BASELINE configs[1]) deflated-norm error per principal vector: GPU mapi_pca_topk vs the fp64 oracle,
end to end, and the same with the GPU fed the oracle's own D_i (fp64 -> one fp32 rounding).  Decides the
norm tolerance of tests/test_gpu_pca.py (reading R8)."""
import numpy as np
import torch

import oracle as orc
import paper_2110_12065_b200 as m
import synth

cfg = synth.cfg2(device="cuda")
A_host = cfg["A"].cpu().numpy()
k, T = cfg["k"], cfg["iters"]
res = m.pca_topk(cfg["A"], k, T, torch.from_numpy(cfg["b0"]).cuda())
ref = orc.pca_topk(A_host, k, T, cfg["b0"])
P = res.P.cpu().numpy()
print("vector  e2e_norm_maxrel  e2e_1-cos  e2e_maxabs  cond_norm_maxrel  cond_1-cos")
b0 = torch.from_numpy(cfg["b0"]).cuda()
for i in range(k):
    ng = res.norms[i].cpu().numpy().astype(np.float64)
    e = np.max(np.abs(ng - ref.norms[i]) / np.abs(ref.norms[i]))
    a, b = P[i].astype(np.float64), ref.P[i]
    cos = abs(a @ b) / np.linalg.norm(a) / np.linalg.norm(b)
    D = orc.deflate(A_host, ref.P, i)
    r = m.iterate(torch.from_numpy(D.astype(np.float32)).cuda(), b0, T)
    rd = orc.mapi(D, cfg["b0"], T)  # fp64 D: the oracle's own trajectory
    ce = np.max(np.abs(r.norms.cpu().numpy() - rd.norms) / np.abs(rd.norms))
    wl = r.w_l2.cpu().numpy().astype(np.float64)
    c2 = abs(wl @ ref.P[i]) / np.linalg.norm(wl)
    print(f"{i:6d}  {e:15.3e}  {1 - cos:9.2e}  {np.max(np.abs(a - b)):10.2e}  {ce:16.3e}  {1 - c2:9.2e}")
