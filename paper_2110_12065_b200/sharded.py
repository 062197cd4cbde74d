"""Row-sharded multi-GPU MAPI.

Rank r of a world of size P holds the contiguous row block [r*n/P, (r+1)*n/P) of A.  Every iteration
of Algorithm 1:

    y_local = A_local (+) w_t              K1 mapi_mavp_matvec on the local rows (HBM-bound, 1/P of A)
    y       = all-gather(y_local)          the one real exchange step: n*4 bytes (128 KiB at cfg3), NCCL
    w_{t+1} = y / ||y||_1, delta_t         mapi_normalize on the FULL y, identical fixed-order kernel on
                                           every rank -> bitwise identical w and stop decision everywhere
                                           (no separate all-reduce of s is needed)

The local mat-vec, the all-gather and the normalisation are injectable so that the orchestration (the
partition, the gather order, the per-rank agreement) is tested with gloo on CPU (tests/test_dist_host.py).
The product path passes the CUDA entry points and torch.distributed over NCCL.
"""
from __future__ import annotations

from dataclasses import dataclass


def row_partition(n: int, world: int, rank: int):
    """Contiguous balanced row block of `rank` (n % world == 0 required by the all-gather layout)."""
    if n % world != 0:
        raise ValueError(f"row-sharded MAPI needs n ({n}) divisible by the world size ({world})")
    per = n // world
    return rank * per, (rank + 1) * per


@dataclass
class ShardedResult:
    w: object
    norms: object
    deltas: object
    iters_done: int


def iterate_sharded(A_local, n: int, b0, iters: int, tol: float = 0.0, op: int = 0, group=None,
                    local_matvec=None, all_gather=None, normalize=None, check_every: int = 0) -> ShardedResult:
    """MAPI on a row-sharded A.  A_local: this rank's (n/P) x n rows; b0: the full start vector.

    local_matvec(A_local, w, y_local), all_gather(y_full, y_local) and normalize(y, w, s_out, delta_out,
    status_out) default to the CUDA library and NCCL.  With tol > 0 the stop test reads delta on the
    host every `check_every` iterations (default every iteration); with tol == 0 the loop never syncs.
    """
    import torch
    import torch.distributed as dist

    from . import MapiError, STATUS
    from . import mavp_matvec as _matvec
    from . import normalize as _normalize

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rows = A_local.shape[0]
    if rows * world != n:
        raise ValueError(f"A_local has {rows} rows; expected n / world = {n // max(world, 1)}")
    dev = A_local.device
    w = b0.clone().to(dev)
    y_local = torch.empty(rows, dtype=torch.float32, device=dev)
    y = torch.empty(n, dtype=torch.float32, device=dev)
    norms = torch.zeros(iters, dtype=torch.float32, device=dev)
    deltas = torch.zeros(iters, dtype=torch.float32, device=dev)
    status = torch.zeros(iters, dtype=torch.int32, device=dev)
    fused = local_matvec is None and normalize is None
    if fused:
        # product path, one kernel + one all-gather per iteration: iteration t's launch normalises the
        # gathered y_{t-1} inside every CTA (mapi_matvec_normalized) and then computes its local rows
        from . import load

        lib = load()
        if A_local.dim() != 2 or A_local.stride(1) != 1:
            raise ValueError("A_local must be a row-major fp32 CUDA tensor")
        sp = torch.cuda.current_stream(dev).cuda_stream
        wbuf = torch.empty(2, n, dtype=torch.float32, device=dev)
        wbuf[0].copy_(w)
        pa, lda, pyl, py = A_local.data_ptr(), A_local.stride(0), y_local.data_ptr(), y.data_ptr()
        pw = [wbuf[0].data_ptr(), wbuf[1].data_ptr()]
        pn, pd, ps = norms.data_ptr(), deltas.data_ptr(), status.data_ptr()

        def fused_step(t):
            if t == 0:  # w_0 = b0 as given: plain mat-vec
                st = lib.mapi_mavp_matvec(op, pa, rows, n, lda, pw[0], pyl, sp)
            else:  # w_t = y_{t-1}/s_{t-1} (recorded as iteration t-1), then y_local = A_local (op) w_t
                st = lib.mapi_matvec_normalized(op, pa, rows, n, lda, py, pw[(t - 1) & 1], pw[t & 1], pyl,
                                                pn + 4 * (t - 1), pd + 4 * (t - 1), ps + 4 * (t - 1), sp)
            if st:
                raise MapiError(st, lib.mapi_last_error_message().decode())

        def final_normalize(t):  # the normalisation of the last gathered y (iteration t)
            tmp = wbuf[t & 1].clone()
            st = lib.mapi_normalize(op, py, n, tmp.data_ptr(), pn + 4 * t, pd + 4 * t, ps + 4 * t, sp)
            if st:
                raise MapiError(st, lib.mapi_last_error_message().decode())
            return tmp
    else:
        local_matvec = local_matvec or (lambda A, w_, yl: _matvec(A, w_, yl, op=op))
        normalize = normalize or (lambda y_, w_, s_, d_, st_: _normalize(y_, w_, s_, d_, st_, op=op))

        def step_normalize(t):
            normalize(y, w, norms[t:t + 1], deltas[t:t + 1], status[t:t + 1])
    if all_gather is None:
        all_gather = (lambda full, part: dist.all_gather_into_tensor(full, part, group=group)) if world > 1 \
            else (lambda full, part: full.copy_(part))
    check_every = check_every or 1
    done = 0
    if fused:
        # the stop test of iteration t is known after launch t+1; a stop at t discards that extra launch's y
        for t in range(iters):
            fused_step(t)
            all_gather(y, y_local)
            if t > 0 and tol > 0.0 and (t % check_every == 0):
                st = int(status[t - 1].item())
                if st != 0:
                    raise MapiError(st, f"{STATUS.get(st, st)} at iteration {t - 1}", t - 1)
                if float(deltas[t - 1].item()) < tol:
                    done = t
                    w = wbuf[t & 1].clone()
                    break
        else:
            w = final_normalize(iters - 1)
            done = iters
    else:
        for t in range(iters):
            local_matvec(A_local, w, y_local)
            all_gather(y, y_local)
            step_normalize(t)
            done = t + 1
            if tol > 0.0 and (done % check_every == 0):
                st = int(status[t].item())
                if st != 0:
                    raise MapiError(st, f"{STATUS.get(st, st)} at iteration {t}", t)
                if float(deltas[t].item()) < tol:
                    break
    st = status[:done].cpu()
    bad = (st != 0).nonzero()
    if bad.numel():
        t = int(bad[0, 0])
        raise MapiError(int(st[t]), f"{STATUS.get(int(st[t]), int(st[t]))} at iteration {t}", t)
    return ShardedResult(w, norms[:done], deltas[:done], done)
