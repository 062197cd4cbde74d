"""Investigation: where the cfg3 end-to-end step time goes (packed symmetric path): H2D of the packed
matrix alone, the device unpack alone, the 100 iterations alone, and the pipelined step."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2110_12065_b200 as m  # noqa: E402
import synth  # noqa: E402


def ev_time(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


m.load()
dev = torch.device("cuda", 0)
cfg = synth.cfg3(device=dev)
A = cfg["A"]
n = A.shape[0]
b0 = torch.from_numpy(cfg["b0"]).to(dev)
t = time.time()
Ap = m.pack_upper(A.cpu(), out=torch.empty(n * (n + 1) // 2, dtype=torch.float32, pin_memory=True))
print(f"host pack {time.time() - t:.1f} s", flush=True)
Ad = torch.empty(n * (n + 1) // 2, dtype=torch.float32, device=dev)
print(f"H2D packed ({Ap.numel() * 4 / 1e9:.2f} GB): {ev_time(lambda: Ad.copy_(Ap, non_blocking=True)):.2f} ms")
Af = torch.empty(n, n, dtype=torch.float32, pin_memory=True)
Af.copy_(A.cpu())
Afd = torch.empty(n, n, dtype=torch.float32, device=dev)
print(f"H2D full ({Af.numel() * 4 / 1e9:.2f} GB): {ev_time(lambda: Afd.copy_(Af, non_blocking=True)):.2f} ms")
print(f"iterate 100 (device-resident): {ev_time(lambda: m.iterate(A, b0, 100)):.2f} ms")
b0h = b0.cpu().pin_memory()
for count in (1, 4):
    ms = ev_time(lambda: m.iterate_host_many_packed([Ap] * count, n, [b0h] * count, 100), reps=1)
    print(f"packed host_many count={count}: {ms:.2f} ms ({ms / count:.2f} per problem)")
    ms = ev_time(lambda: m.iterate_host_many([Af] * count, [b0h] * count, 100), reps=1)
    print(f"full host_many count={count}: {ms:.2f} ms ({ms / count:.2f} per problem)")
