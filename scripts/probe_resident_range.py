"""Investigation: K2r (resident) vs the other dense iteration kernels across n (us / iteration, 200
iterations, events around mapi_iterate, A device-resident).  Used to set the K2r dispatch range."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_12065_b200 as m  # noqa: E402

m.load()
T = 200
for n in [520, 768, 1024, 1536, 2048, 2560, 3072, 3584, 4096]:
    r = np.random.default_rng(n)
    A = torch.from_numpy((r.standard_normal((n, n)) + np.diag(np.abs(r.standard_normal(n)) * 4)).astype(np.float32)).cuda()
    b0 = torch.full((n,), 1.0 / np.sqrt(n), device="cuda")
    row = [f"n={n:5d}"]
    for path in ["resident", "bulk", "rows", "cluster_smem", ""]:
        os.environ["MAPI_DENSE_PATH"] = path
        try:
            m.iterate(A, b0, T)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                m.iterate(A, b0, T)
            e1.record()
            torch.cuda.synchronize()
            row.append(f"{path or 'default'} {1e3 * e0.elapsed_time(e1) / (3 * T):6.2f}")
        except Exception as ex:  # a forced path that cannot run
            row.append(f"{path} ERR {ex}")
    print(" | ".join(row), flush=True)
