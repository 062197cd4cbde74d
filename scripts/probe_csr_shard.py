"""cfg5 through the sharded ranking (K3n) on ONE GPU: per-iteration time of a rank's three steps for worlds of
1, 2, 4, 8 (the rank-0 block of each partition, its exchange replaced by nothing: timing of the local work
only), beside mapi_rank_csr (K3) and mapi_rank_csr_plan (K3s) on the whole graph."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_12065_b200 as m
import synth
from paper_2110_12065_b200 import sharded

c = synth.cfg5()
n = c["n"]
rp = torch.from_numpy(np.ascontiguousarray(c["row_ptr"])).to(torch.int32).cuda()
ci = torch.from_numpy(np.ascontiguousarray(c["col_idx"]).astype(np.int32)).cuda()
b0 = torch.from_numpy(c["b0"]).cuda()
cap, bg = m.csr_prepare(n, rp, ci, 0.85)
iters = 50


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


t = timed(lambda: m.rank_csr(n, rp, ci, cap, bg, b0, iters, 0.0))
print(f"K3  mapi_rank_csr       whole graph: {1e3 * t / iters:8.1f} us / iteration")
plan = m.csr_plan(n, rp, ci)
t = timed(lambda: m.rank_csr_plan(plan, cap, bg, b0, iters, 0.0))
print(f"K3s mapi_rank_csr_plan  whole graph: {1e3 * t / iters:8.1f} us / iteration")
for world in (1, 2, 4, 8):
    starts = sharded.csr_row_partition(c["row_ptr"], world)
    for rank in sorted({0, world - 1}):
        r0, r1 = starts[rank], starts[rank + 1]
        rpl, cil = sharded.csr_shard(rp, ci, r0, r1)
        ses = sharded.CsrShardSession(n, r0, rpl, cil, cap, bg, b0, iters, 0.0)

        def run():
            ses.begin()
            for it in range(iters):
                ses.rows(it)
                ses.normalize(it)

        t = timed(run)

        def rows_only():
            for it in range(iters):
                ses.rows(it)

        tr = timed(rows_only)
        print(f"K3n world {world} rank {rank}: rows [{r0}, {r1}) {cil.numel():>9d} edges: {1e3 * t / iters:8.1f} us / iteration "
              f"(rows {1e3 * tr / iters:7.1f} us, node kernels {1e3 * (t - tr) / iters:6.1f} us); exchange bytes in: "
              f"{4 * (n - (r1 - r0)) / 1e6:.1f} MB")
