"""Exercise every libmapi entry point on small inputs (for compute-sanitizer memcheck / racecheck /
synccheck / initcheck runs).  Small shapes with ragged tails; exits non-zero on error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2110_12065_b200 as m
import synth

m.load()
dev = "cuda"
r = np.random.default_rng(0)
# dense: matvec (smem / global x), iterate on every path, host variant, pca
for shape in ((33, 257), (5, 60001)):
    M, _ = synth.random_matrix(*shape, seed=1, lda=shape[1] + 3)
    m.mavp_matvec(torch.from_numpy(M).to(dev)[:, : shape[1]], torch.from_numpy(synth.random_vector(shape[1], 2)).to(dev))
for n, path in ((300, "cluster"), (300, "rows"), (8200, "coop"), (300, "multi"), (1000, "rows")):
    os.environ["MAPI_DENSE_PATH"] = path
    A = torch.from_numpy((r.standard_normal((n, n)) + np.eye(n) * 3).astype(np.float32)).to(dev)
    b0 = torch.full((n,), 1.0 / np.sqrt(n), device=dev)
    for op in (0, 1, 2):
        m.iterate(A, b0, 4, tol=1e-9, op=op)
os.environ.pop("MAPI_DENSE_PATH")
A = torch.from_numpy((r.standard_normal((300, 300)) + np.eye(300) * 3).astype(np.float32))
m.iterate_host(A.pin_memory(), torch.full((300,), 0.05).pin_memory(), 3)
C = torch.from_numpy(synth.covariance_like(r.standard_normal((257, 300)), 1 / 300)).to(dev)
m.pca_topk(C, 3, 5, torch.full((257,), 1 / np.sqrt(257), device=dev))
# batched: every kernel
for path in ("v1", "v2", "v3"):
    os.environ["MAPI_BATCHED_PATH"] = path
    A = torch.from_numpy((r.standard_normal((260, 260)) + np.eye(260) * 3).astype(np.float32)).to(dev)
    m.iterate_batched(A, torch.from_numpy(r.standard_normal((70, 260)).astype(np.float32)).to(dev), 3)
os.environ.pop("MAPI_BATCHED_PATH")
# ranking
g = synth.gnutella_like()
rp = torch.from_numpy(g["row_ptr"].astype(np.int32)).to(dev)
ci = torch.from_numpy(g["col_idx"]).to(dev)
cap, bg = m.csr_prepare(g["n"], rp, ci)
m.rank_csr(g["n"], rp, ci, cap, bg, torch.from_numpy(g["b0"]).to(dev), 5, 0.0)
# matmat (16 B and 4 B staging), NEXT-2
for K in (12, 10):
    V = torch.from_numpy(r.standard_normal((300, K)).astype(np.float32)).to(dev)
    m.min_covariance(V)
Vraw, _ = synth.occluded_copies(D=32, N=5, seed=2, tile=8)
Vd = torch.from_numpy(Vraw).to(dev)
Vc, _ = m.center_rows(Vd)
Cm = m.min_covariance(Vc)
w = m.iterate(Cm, torch.full((1024,), 1 / 32.0, device=dev), 10).w
D = m.mavp_deflate(Cm, w)
m.mavp_reconstruct(torch.stack([w, w], 1).contiguous(), Vd)
torch.cuda.synchronize()
print("sanitize_small: all entry points ran, launches =", m.launch_count())
