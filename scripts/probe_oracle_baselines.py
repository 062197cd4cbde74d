"""BASELINE.md §3 oracle timings on the GPU box's host (test infrastructure; the oracle is a reported
baseline, not the target): the host (nproc, CPU model, NUMA), cfg1 and cfg2 on all threads and on ONE thread
(cfg2 with the deflation builds broken out), and the cfg3 sample policies of both bench legs in one process
(1-iteration calls vs one k-iteration call) to explain their gap."""
import os
import subprocess
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402


def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=30).stdout.strip()
    except Exception as e:  # noqa: BLE001
        return f"({e})"


oracle.build()
allt = oracle.num_threads()
print("nproc", sh("nproc"), "| oracle OpenMP threads", allt)
print("cpu", sh("lscpu | grep -E 'Model name|Socket|NUMA node\\(s\\)|Thread\\(s\\) per core' | tr -s ' '"))
for threads in (allt, 1):
    oracle.set_num_threads(threads)
    c1 = synth.cfg1()
    t0 = time.perf_counter()
    r = oracle.mapi(c1["A"], c1["b0"].astype(np.float64), c1["iters"])
    dt = time.perf_counter() - t0
    print(f"cfg1 threads={threads}: {r.iters_done} iterations in {dt * 1e3:.2f} ms = {r.iters_done / dt:.1f} it/s")
    c2 = synth.cfg2()
    C, b0, k, iters = c2["C"] if "C" in c2 else c2["A"], c2["b0"].astype(np.float64), c2.get("k", 8), c2["iters"]
    t0 = time.perf_counter()
    res = oracle.pca_topk(C, k, iters, b0)
    dt = time.perf_counter() - t0
    # the deflation builds alone (D_i for i = 1..k-1 from the computed vectors)
    t1 = time.perf_counter()
    for i in range(1, k):
        oracle.deflate(C, res.P, i)
    dd = time.perf_counter() - t1
    tot = int(np.sum(res.iters_done)) if hasattr(res.iters_done, "__len__") else k * iters
    print(f"cfg2 threads={threads}: top-{k} x {iters} iterations incl. deflation in {dt:.2f} s = {tot / dt:.2f} it/s; "
          f"the {k - 1} deflation builds alone {dd:.2f} s")
oracle.set_num_threads(allt)
try:
    import torch

    dev = "cuda" if torch.cuda.is_available() else None
except Exception:  # noqa: BLE001
    dev = None
c3 = synth.cfg3(device=dev)
A = c3["A"].cpu().numpy() if dev else c3["A"]
b0 = c3["b0"].astype(np.float64)
per = []
for _ in range(4):
    t0 = time.perf_counter()
    oracle.mapi(A, b0, 1)
    per.append(time.perf_counter() - t0)
print("cfg3 reference-arm policy (1-iteration calls): s/iteration", " ".join(f"{x:.3f}" for x in per))
t0 = time.perf_counter()
r = oracle.mapi(A, b0, 8)
dt = time.perf_counter() - t0
print(f"cfg3 repo-arm policy (one 8-iteration call): {dt / 8:.3f} s/iteration = {8 / dt:.2f} it/s")
A2 = np.array(A, copy=True)  # a second copy, first-touched by numpy in one thread
t0 = time.perf_counter()
oracle.mapi(A2, b0, 2)
print(f"cfg3 on a fresh single-thread-touched copy: {(time.perf_counter() - t0) / 2:.3f} s/iteration")
