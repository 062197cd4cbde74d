"""Algorithm 3 (mini-batch MAPI with momentum) at the paper's shape on the host: the fp64 oracle's
time per iteration (is a GPU path worth building?) and the alignment with u1 on the paper's synthetic
eigen-gap data for both gram readings (R14), beta and batch sizes.  Test infrastructure only."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402

oracle.build()
r = np.random.default_rng(0)
N, D = 10**6, 10
X = r.standard_normal((N, D))
for s in (128, 1024):
    idx = r.integers(0, N, (100, s))
    w0 = r.standard_normal(D)
    w0 /= np.linalg.norm(w0)
    oracle.minibatch_mapi(X, idx, 0.225, w0)
    t0 = time.perf_counter()
    oracle.minibatch_mapi(X, idx, 0.225, w0)
    dt = time.perf_counter() - t0
    print(f"N=1e6 D=10 s={s} T=100: {dt * 1e3:.2f} ms ({dt * 1e4:.1f} us/iteration, {s * D * D + D * D} MAVP terms/iteration)")


def dataset(N, D=10, gap=0.1, seed=0):  # X = U Sigma V^T, Sigma = diag(1, sqrt(0.9), ...)
    g = np.random.default_rng(seed)
    U, _ = np.linalg.qr(g.standard_normal((N, D)))
    V, _ = np.linalg.qr(g.standard_normal((D, D)))
    sig = np.array([1.0] + [np.sqrt(1 - gap)] * (D - 1))
    return (U * sig) @ V.T, V[:, 0]


X, u1 = dataset(10**5)
g = np.random.default_rng(1)
for gram in ("min1", "dot"):
    for beta in (0.0, 0.225):
        for s in (128, 1024):
            idx = g.integers(0, X.shape[0], (100, s))
            w0 = g.standard_normal(10)
            w0 /= np.linalg.norm(w0)
            w = oracle.minibatch_mapi(X, idx, beta, w0, gram=gram).w_l2
            print(f"N=1e5 gram={gram} beta={beta} s={s}: alignment error 1-(w.u1)^2 = {1 - (w @ u1) ** 2:.3f}")
