"""Per-iteration latency of the dense iteration kernels for small n (investigation only):
kernel time (CUDA events around the launch) for T = 1, 11, 51, 201 iterations per dense path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2110_12065_b200 as m
import synth

m.load()
for n in (256, 512, 4096):
    if n == 256:
        A = torch.from_numpy(synth.cfg1()["A"]).cuda()
    else:
        r = np.random.default_rng(0)
        A = torch.from_numpy((r.standard_normal((n, n)) + np.eye(n) * 5).astype(np.float32)).cuda()
    b0 = torch.full((n,), 1.0 / np.sqrt(n), device="cuda")
    for path in ("cluster", "rows", "coop"):
        os.environ["MAPI_DENSE_PATH"] = path
        m.set_profiling(True)
        res = {}
        for T in (1, 11, 51, 201):
            best = 1e9
            for _ in range(5):
                m.iterate(A, b0, T, want_trace=False)
                best = min(best, m.last_kernel_ms())
            res[T] = best
        per = (res[201] - res[11]) / 190 * 1e3
        print(f"n={n:5d} path={path:8s} T=1 {res[1]*1e3:8.1f} us  T=51 {res[51]*1e3:8.1f} us  "
              f"per-iteration {per:6.2f} us")
