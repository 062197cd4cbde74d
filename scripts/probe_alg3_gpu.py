"""Alg. 3 on the GPU vs the fp64 oracle: per-iteration norm differences (error growth of the stochastic
iteration in fp32) and the time per call at the paper's shape.  Test infrastructure only."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
import paper_2110_12065_b200 as m
oracle.build()
X, _ = synth.stochastic_pca(N=100_000, D=10, seed=7)
X = (X * np.float32(np.sqrt(X.shape[0]))).astype(np.float32)
for s, beta in ((128, 0.0), (128, 0.225), (1024, 0.0)):
    idx = synth.batch_draws(X.shape[0], 100, s, seed=8)
    w = np.random.default_rng(1).standard_normal(10); w0 = (w / np.linalg.norm(w)).astype(np.float32)
    ref = oracle.minibatch_mapi(X.astype(np.float64), idx.astype(np.int64), beta, w0.astype(np.float64))
    Xd, id_, w0d = torch.from_numpy(X).cuda(), torch.from_numpy(idx).cuda(), torch.from_numpy(w0).cuda()
    res = m.minibatch(Xd, id_, beta, w0d)
    rel = np.abs(res.norms.cpu().numpy() - ref.norms) / ref.norms
    print(f"s={s} beta={beta}: norm rel err at t=0,1,2,5,10,20,50,99:", " ".join(f"{rel[t]:.1e}" for t in (0, 1, 2, 5, 10, 20, 50, 99)),
          "cos", abs(float(np.dot(res.w_l2.cpu().numpy().astype(np.float64), ref.w_l2))))
    for T in (1, 2, 5, 10):
        r2 = oracle.minibatch_mapi(X.astype(np.float64), idx[:T].astype(np.int64), beta, w0.astype(np.float64))
        g2 = m.minibatch(Xd, id_[:T].contiguous(), beta, w0d)
        print(f"   T={T}: max|dw_l2| {np.max(np.abs(g2.w_l2.cpu().numpy() - r2.w_l2)):.2e}")
# timing at the paper's shape (N = 1e6)
X, _ = synth.stochastic_pca(N=1_000_000, D=10, seed=7)
Xd = torch.from_numpy(X).cuda()
for s in (128, 1024):
    id_ = torch.from_numpy(synth.batch_draws(X.shape[0], 100, s, seed=8)).cuda()
    for _ in range(3): m.minibatch(Xd, id_, 0.225, w0d)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(20): m.minibatch(Xd, id_, 0.225, w0d)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 20
    print(f"N=1e6 D=10 s={s} T=100: {dt*1e3:.3f} ms per call ({dt*1e4:.2f} us/iteration)")
