"""Per-iteration slope and fixed cost of mapi_iterate (kernel events) at mid n, per dense path
(investigation only): the cfg2 matrix (n = 4096) and random ones at other n."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2110_12065_b200 as m
import synth

m.load()
m.set_profiling(True)
sizes = [int(x) for x in os.environ.get("PROBE_SIZES", "1024,2048,4096,6144,8192,16384").split(",")]
mats = {}
if 4096 in sizes:
    mats[4096] = synth.cfg2(device="cuda")["A"]
if 256 in sizes:
    mats[256] = torch.from_numpy(synth.cfg1()["A"]).cuda()
for n in [x for x in sizes if x not in (256, 4096)]:
    r = np.random.default_rng(n)
    mats[n] = torch.from_numpy((r.standard_normal((n, n)) + np.eye(n) * 5).astype(np.float32)).cuda()
for n, A in sorted(mats.items()):
    b0 = torch.full((n,), 1.0 / np.sqrt(n), device="cuda")
    for path in os.environ.get("PROBE_PATHS", "rows,bulk,coop").split(","):
        os.environ["MAPI_DENSE_PATH"] = path
        res = {}
        for T in (1, 11, 101):
            best = 1e9
            for _ in range(5):
                m.iterate(A, b0, T, want_trace=False)
                best = min(best, m.last_kernel_ms())
            res[T] = best
        slope = (res[101] - res[11]) / 90 * 1e3
        gbs = n * n * 4 / (slope * 1e-6) / 1e9
        print(f"n {n:6d} {path:5s} T=1 {res[1]*1e3:8.1f} us  T=101 {res[101]*1e3:9.1f} us  slope {slope:7.2f} us/it  {gbs:7.0f} GB/s", flush=True)
