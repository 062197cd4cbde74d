"""Investigation: small-n dense kernels (K6t single CTA, K6r cluster, default) in us / iteration (50 and
500 iterations per call, events around mapi_iterate, A device-resident)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_12065_b200 as m  # noqa: E402

m.load()
for n in [64, 128, 200, 256, 384, 512]:
    r = np.random.default_rng(n)
    A = torch.from_numpy((r.standard_normal((n, n)) + np.diag(np.abs(r.standard_normal(n)) * 4)).astype(np.float32)).cuda()
    b0 = torch.full((n,), 1.0 / np.sqrt(n), device="cuda")
    row = [f"n={n:4d}"]
    for T in (50, 500):
        for path in ["single", "cluster", ""]:
            os.environ["MAPI_DENSE_PATH"] = path
            m.iterate(A, b0, T)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                m.iterate(A, b0, T)
            e1.record()
            torch.cuda.synchronize()
            row.append(f"T={T} {path or 'default'} {1e3 * e0.elapsed_time(e1) / (5 * T):6.2f}")
    print(" | ".join(row), flush=True)
