"""Row-sharded multi-GPU MAPI.

Rank r of a world of size P holds the contiguous row block [r*n/P, (r+1)*n/P) of A.  Every iteration
of Algorithm 1:

    y_local = A_local (+) w_t              K1 mapi_mavp_matvec on the local rows (HBM-bound, 1/P of A)
    y       = all-gather(y_local)          the one real exchange step: n*4 bytes (128 KiB at cfg3), NCCL
    w_{t+1} = y / ||y||_1, delta_t         mapi_normalize on the FULL y, identical fixed-order kernel on
                                           every rank -> bitwise identical w and stop decision everywhere
                                           (no separate all-reduce of s is needed)

`iterate_batched_sharded` partitions the k independent runs of the batched path (cfg4) over the ranks — no
data-path collective at all.

The local mat-vec, the all-gather and the normalisation are injectable so that the orchestration (the
partition, the gather order, the per-rank agreement) is tested with gloo on CPU (tests/test_dist_host.py).
The product path passes the CUDA entry points and torch.distributed over NCCL.

`P2PExchange` + `iterate_sharded_p2p` / `iterate_sym_sharded_p2p` are the fused paths (K2p / K2sp,
csrc/p2p.cuh): ONE cooperative launch per rank runs every iteration and the exchange happens inside it —
each rank stores its share straight into every rank's exchange buffer over NVLink (CUDA IPC mappings),
then one thread release-adds every rank's arrival flag at system scope and all CTAs wait for all of them;
no NCCL call on the data path.  K2sp (the N > 1 default for symmetric A) splits K2s's upper-triangle task
list over the ranks and exchanges partial y vectors.  The host side here only sets up the mappings once
(IPC handles and SM counts all-gathered over torch.distributed) and carries the global iteration epoch /
flag base from call to call.
"""
from __future__ import annotations

from dataclasses import dataclass


def row_partition(n: int, world: int, rank: int):
    """Contiguous balanced row block of `rank` (n % world == 0 required by the all-gather layout)."""
    if n % world != 0:
        raise ValueError(f"row-sharded MAPI needs n ({n}) divisible by the world size ({world})")
    per = n // world
    return rank * per, (rank + 1) * per


def vector_partition(k: int, world: int, rank: int):
    """Contiguous balanced slice [k0, k1) of k independent start vectors for `rank` (k need not divide)."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside a world of {world}")
    return rank * k // world, (rank + 1) * k // world


def iterate_batched_sharded(A, B0, iters: int, tol: float = 0.0, op: int = 0, group=None, run_local=None,
                            gather: bool = False):
    """Batched MAPI (P:69-70 with p = k columns, BASELINE configs[3]) over the ranks: the k runs are
    independent problems on the same A, so they partition with NO data-path collective: every
    rank holds A (1 GiB at cfg4) and runs its contiguous slice of the start vectors through
    mapi_iterate_batched.  B0: the FULL k x n starts (every rank slices its own rows).  Returns (k0, k1,
    result) with the local slice's BatchedResult, or, with gather=True, every rank's W / norms / iteration
    counts all-gathered afterwards (one collective after the run, off the hot path; needs k % world == 0).
    run_local(A, B0_local, iters, tol, op) is injectable for the CPU (gloo) test."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    k = B0.shape[0]
    k0, k1 = vector_partition(k, world, rank)
    if run_local is None:
        from . import iterate_batched as run_local
    res = run_local(A, B0[k0:k1].contiguous(), iters, tol, op) if k1 > k0 else None
    if not gather or world == 1:
        return k0, k1, res
    if k % world != 0:
        raise ValueError(f"gather=True needs k ({k}) divisible by the world size ({world})")
    W = torch.empty_like(B0)
    dist.all_gather_into_tensor(W, res.W.contiguous(), group=group)
    T_, kl = res.norms.shape
    norms = torch.empty((world * T_, kl), dtype=res.norms.dtype, device=res.norms.device)
    dist.all_gather_into_tensor(norms, res.norms.contiguous(), group=group)
    norms = norms.view(world, T_, kl)
    done = torch.tensor(list(res.iters_done), dtype=torch.int32, device=B0.device)
    done_all = torch.empty(k, dtype=torch.int32, device=B0.device)
    dist.all_gather_into_tensor(done_all, done, group=group)
    # norms are iters x k_local per rank: back to iters x k, vector-major as on one GPU
    return k0, k1, (W, torch.cat(list(norms), dim=1), done_all)


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


# ------------------------------------------------------------------------------ fused P2P exchange (K2p)


class P2PExchange:
    """The per-rank exchange buffer of K2p / K2sp and its peers' IPC mappings.

    lib: the loaded libmapi (or a stand-in with the same six entry points, for host-logic tests);
    allgather(bytes) -> list of every rank's bytes, in rank order (torch.distributed by default).
    `grid` is the CTA count every rank launches with: the minimum of the ranks' SM counts (`sms`, default:
    the device's), agreed here once, because the kernels' row ownership and summation orders depend on it.
    `epoch` / `flag_base` carry the global iteration index and the own flag value across calls; they
    advance by `published` and `published * world` after each call (one arrival per rank per iteration),
    identically on every rank.
    """

    def __init__(self, n: int, rank: int, world: int, lib=None, allgather=None, group=None, device=None,
                 sms: int = None):
        import ctypes

        if lib is None:
            from . import load

            lib = load()
        self.lib, self.n, self.rank, self.world = lib, n, rank, world
        self.bytes = int(lib.mapi_p2p_exchange_bytes(n, world))
        if allgather is None:
            allgather = _dist_allgather_bytes(group, device)
        if sms is None:
            import torch

            sms = torch.cuda.get_device_properties(device if device is not None else 0).multi_processor_count
        counts = [int.from_bytes(b, "little") for b in allgather(int(sms).to_bytes(8, "little"))]
        if len(counts) != world:
            raise ValueError(f"expected {world} SM counts, got {len(counts)}")
        self.grid = min(min(counts), 1024)
        ptr = ctypes.c_void_p()
        self._check(lib.mapi_p2p_alloc(self.bytes, ctypes.byref(ptr)))
        self.own = int(ptr.value)
        handle = ctypes.create_string_buffer(64)
        self._check(lib.mapi_ipc_get_handle(self.own, handle))
        handles = allgather(bytes(handle.raw))
        if len(handles) != world:
            raise ValueError(f"expected {world} handles, got {len(handles)}")
        self.opened = []
        peers = []
        for q, h in enumerate(handles):
            if q == rank:
                peers.append(self.own)
                continue
            out = ctypes.c_void_p()
            self._check(lib.mapi_ipc_open_handle(ctypes.create_string_buffer(h, 64), ctypes.byref(out)))
            self.opened.append(int(out.value))
            peers.append(int(out.value))
        self.peer_addrs = peers
        self.epoch = 0
        self.flag_base = 0
        self.peers_dev = None
        if device is not None:
            import torch

            self.peers_dev = torch.tensor(peers, dtype=torch.int64, device=device)

    def _check(self, st):
        if st:
            from . import MapiError

            raise MapiError(st, self.lib.mapi_last_error_message().decode(errors="replace"))

    def advance(self, published: int):
        self.epoch += published
        self.flag_base += published * self.world

    def close(self):
        for a in self.opened:
            self.lib.mapi_ipc_close_handle(a)
        self.opened = []
        if self.own:
            self.lib.mapi_p2p_free(self.own)
            self.own = 0


def _dist_allgather_bytes(group, device):
    import torch
    import torch.distributed as dist

    def gather(b: bytes):
        if not dist.is_initialized() or dist.get_world_size(group) == 1:
            return [b]
        t = torch.frombuffer(bytearray(b), dtype=torch.uint8).to(device if device is not None else "cpu")
        out = torch.empty(dist.get_world_size(group) * t.numel(), dtype=torch.uint8, device=t.device)
        dist.all_gather_into_tensor(out, t, group=group)
        return [bytes(c.cpu().numpy().tobytes()) for c in out.view(-1, t.numel())]

    return gather


def iterate_sharded_p2p(A_local, n: int, row0: int, b0, iters: int, exchange: P2PExchange, tol: float = 0.0,
                        op: int = 0, want_trace: bool = True) -> ShardedResult:
    """MAPI on a row-sharded A with the exchange fused into one persistent kernel per rank (K2p)."""
    import ctypes

    import torch

    from . import MapiError, WS_ITERATE_SHARDED

    lib = exchange.lib
    dev = A_local.device
    m = A_local.shape[0]
    if A_local.dim() != 2 or A_local.stride(1) != 1 or A_local.dtype != torch.float32:
        raise ValueError("A_local must be a row-major fp32 CUDA tensor")
    if exchange.peers_dev is None:
        exchange.peers_dev = torch.tensor(exchange.peer_addrs, dtype=torch.int64, device=dev)
    w = torch.empty(n, dtype=torch.float32, device=dev)
    norms = torch.zeros(iters, dtype=torch.float32, device=dev) if want_trace else None
    deltas = torch.zeros(iters, dtype=torch.float32, device=dev) if want_trace else None
    ws = torch.empty(int(lib.mapi_workspace_size(WS_ITERATE_SHARDED, 0, 0, 0)), dtype=torch.uint8, device=dev)
    done, published, grid = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
    sp = torch.cuda.current_stream(dev).cuda_stream
    st = lib.mapi_iterate_sharded(op, A_local.data_ptr(), m, n, A_local.stride(0), row0, b0.data_ptr(), iters,
                                  float(tol), exchange.rank, exchange.world, exchange.peers_dev.data_ptr(),
                                  exchange.epoch, exchange.flag_base, exchange.grid, w.data_ptr(),
                                  None if norms is None else norms.data_ptr(),
                                  None if deltas is None else deltas.data_ptr(), ctypes.byref(done),
                                  ctypes.byref(published), ctypes.byref(grid), ws.data_ptr(), ws.numel(), sp)
    exchange.advance(published.value)
    if st:
        raise MapiError(st, lib.mapi_last_error_message().decode(errors="replace"), done.value)
    k = done.value
    return ShardedResult(w, norms[:k] if norms is not None else None, deltas[:k] if deltas is not None else None, k)


# ------------------------------------------------------------------------------ sharded symmetric (K2sp)


def sym_shard(n: int, rank: int, world: int, lib=None):
    """(row_lo, row_hi, task_lo, task_hi) of `rank` for K2sp: the contiguous slice of K2s's upper-triangle
    task list it runs and the rows those tasks read (mapi_sym_shard_rows; host-only arithmetic)."""
    import ctypes

    if lib is None:
        from . import load

        lib = load()
    out = [ctypes.c_int64() for _ in range(4)]
    st = lib.mapi_sym_shard_rows(n, rank, world, *[ctypes.byref(o) for o in out])
    if st:
        from . import MapiError

        raise MapiError(st, lib.mapi_last_error_message().decode(errors="replace"))
    return tuple(int(o.value) for o in out)


def iterate_sym_sharded_p2p(A_local, row_lo: int, row_hi: int, n: int, b0, iters: int, exchange: P2PExchange,
                            tol: float = 0.0, op: int = 0, want_trace: bool = True, ws=None) -> ShardedResult:
    """MAPI on a symmetric A whose upper-triangle task list is split over the ranks (K2sp,
    mapi_iterate_sym_sharded): A_local holds rows [row_lo, row_hi) = sym_shard(n, rank, world)[:2] (full
    rows; only their upper-triangle part is read).  Every rank returns the same full w."""
    import ctypes

    import torch

    from . import MapiError, WS_ITERATE_SYM

    lib = exchange.lib
    dev = A_local.device
    if A_local.dim() != 2 or A_local.stride(1) != 1 or A_local.dtype != torch.float32:
        raise ValueError("A_local must be a row-major fp32 CUDA tensor")
    if A_local.shape[0] != row_hi - row_lo:
        raise ValueError(f"A_local has {A_local.shape[0]} rows; the shard holds {row_hi - row_lo}")
    if exchange.peers_dev is None:
        exchange.peers_dev = torch.tensor(exchange.peer_addrs, dtype=torch.int64, device=dev)
    w = torch.empty(n, dtype=torch.float32, device=dev)
    norms = torch.zeros(iters, dtype=torch.float32, device=dev) if want_trace else None
    deltas = torch.zeros(iters, dtype=torch.float32, device=dev) if want_trace else None
    need = int(lib.mapi_workspace_size(WS_ITERATE_SYM, n, 0, 0))
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
    done, published, grid = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
    sp = torch.cuda.current_stream(dev).cuda_stream
    st = lib.mapi_iterate_sym_sharded(op, A_local.data_ptr(), row_lo, row_hi, n, A_local.stride(0), b0.data_ptr(),
                                      iters, float(tol), exchange.rank, exchange.world,
                                      exchange.peers_dev.data_ptr(), exchange.epoch, exchange.flag_base,
                                      exchange.grid, w.data_ptr(), None if norms is None else norms.data_ptr(),
                                      None if deltas is None else deltas.data_ptr(), ctypes.byref(done),
                                      ctypes.byref(published), ctypes.byref(grid), ws.data_ptr(), ws.numel(), sp)
    exchange.advance(published.value)
    if st:
        raise MapiError(st, lib.mapi_last_error_message().decode(errors="replace"), done.value)
    k = done.value
    return ShardedResult(w, norms[:k] if norms is not None else None, deltas[:k] if deltas is not None else None, k)


# --------------------------------------------------------------- CSR ranking over ranks (K3n)


def csr_row_partition(row_ptr, world: int):
    """Contiguous destination-row blocks [starts[r], starts[r+1]) of near-equal merge-path cost
    (rows + in-edges: what the gather kernel's tiles count), from the host copy of row_ptr (n + 1).  Index
    bookkeeping only — no method arithmetic.  Returns world + 1 ints; blocks may be empty when world > n."""
    import numpy as np

    rp = np.asarray(row_ptr.cpu() if hasattr(row_ptr, "cpu") else row_ptr, dtype=np.int64)
    n = rp.shape[0] - 1
    if world < 1:
        raise ValueError("world must be >= 1")
    cost = rp - rp[0] + np.arange(n + 1, dtype=np.int64)  # items before row i
    total = int(cost[-1])
    starts = [0]
    for r in range(1, world):
        starts.append(max(starts[-1], int(np.searchsorted(cost, (total * r + world - 1) // world, side="left"))))
    starts.append(n)
    return [min(s, n) for s in starts]


def csr_shard(row_ptr, col_idx, r0: int, r1: int):
    """The sub-CSR of the destination rows [r0, r1): row_ptr rebased to 0 (r1 - r0 + 1 entries) and the
    matching slice of col_idx (global source ids kept)."""
    lo, hi = int(row_ptr[r0]), int(row_ptr[r1])
    return (row_ptr[r0:r1 + 1] - lo).contiguous(), col_idx[lo:hi].contiguous()


class CsrShardSession:
    """One rank's run of the sharded ranking (mapi_rank_csr_shard_*): begin() once, then per iteration
    rows(t) -> the caller's all-gather of the e_t blocks -> normalize(t); finish() returns the result.
    Everything is enqueued on the current stream.  `lib` is injectable for the CPU orchestration test."""

    def __init__(self, n: int, row0: int, row_ptr_local, col_idx_local, cap, bg, b0, max_iters: int,
                 tol: float = 1e-7, lib=None, stream=None):
        import ctypes

        import torch

        from . import WS_RANK_CSR_SHARD, load

        self.lib = lib or load()
        self.n, self.row0, self.m = int(n), int(row0), int(row_ptr_local.numel()) - 1
        self.nnz = int(col_idx_local.numel())
        self.rp, self.ci, self.cap, self.bg, self.b0 = row_ptr_local, col_idx_local, cap, bg, b0
        self.max_iters, self.tol = int(max_iters), float(tol)
        dev = b0.device
        self.need = int(self.lib.mapi_workspace_size(WS_RANK_CSR_SHARD, self.n, self.nnz, self.m))
        self.ws = torch.empty(self.need, dtype=torch.uint8, device=dev)
        self.deltas = torch.zeros(self.max_iters, dtype=torch.float32, device=dev)
        self.sp = stream if stream is not None else (torch.cuda.current_stream(dev).cuda_stream
                                                     if dev.type == "cuda" else None)
        self._c, self._torch = ctypes, torch
        self._e_addr = [0, 0]

    def _check(self, st):
        if st:
            from . import MapiError

            raise MapiError(st, self.lib.mapi_last_error_message().decode())

    def begin(self):
        self._check(self.lib.mapi_rank_csr_shard_begin(self.n, self.m, self.nnz, self.rp.data_ptr(),
                                                       self.cap.data_ptr(), self.bg.data_ptr(), self.b0.data_ptr(),
                                                       self.ws.data_ptr(), self.need, self.sp))

    def rows(self, t: int) -> int:
        """Enqueue iteration t's gather over the owned rows; returns the device address of e_t (n floats)."""
        e = self._c.c_void_p(0)
        self._check(self.lib.mapi_rank_csr_shard_rows(self.n, self.m, self.row0, self.nnz, self.rp.data_ptr(),
                                                      self.ci.data_ptr() if self.nnz else None, int(t),
                                                      self._c.byref(e), self.ws.data_ptr(), self.need, self.sp))
        self._e_addr[t & 1] = e.value
        return e.value

    def e_view(self, t: int):
        """e_t as a tensor view into the workspace (the collective's in-place buffer), at the address
        rows(t) reported."""
        addr = self._e_addr[t & 1]
        if not addr:
            raise RuntimeError("e_view(t) needs rows(t) first")
        base = addr - self.ws.data_ptr()
        if base < 0 or base + 4 * self.n > self.need:
            raise RuntimeError("e_t lies outside the workspace")
        return self.ws[base:base + 4 * self.n].view(self._torch.float32)

    def normalize(self, t: int):
        self._check(self.lib.mapi_rank_csr_shard_normalize(self.n, self.m, self.nnz, self.cap.data_ptr(),
                                                           self.bg.data_ptr(), self.b0.data_ptr(), int(t), self.tol,
                                                           self.deltas.data_ptr(), self.ws.data_ptr(), self.need,
                                                           self.sp))

    def poll(self):
        """(iterations done, stopped) — synchronises the stream (the host's periodic stop check)."""
        done, stopped = self._c.c_int32(0), self._c.c_int32(0)
        self._check(self.lib.mapi_rank_csr_shard_finish(self.n, self.m, self.nnz, None, None, None,
                                                        self._c.byref(done), self._c.byref(stopped),
                                                        self.ws.data_ptr(), self.need, self.sp))
        return done.value, bool(stopped.value)

    def finish(self, want_l2: bool = True):
        from . import IterResult

        dev = self.b0.device
        w = self._torch.empty(self.n, dtype=self._torch.float32, device=dev)
        wl2 = self._torch.empty(self.n, dtype=self._torch.float32, device=dev) if want_l2 else None
        done = self._c.c_int32(0)
        st = self.lib.mapi_rank_csr_shard_finish(self.n, self.m, self.nnz, self.b0.data_ptr(), w.data_ptr(),
                                                 wl2.data_ptr() if want_l2 else None, self._c.byref(done), None,
                                                 self.ws.data_ptr(), self.need, self.sp)
        if st:
            from . import MapiError

            raise MapiError(st, self.lib.mapi_last_error_message().decode(), done.value)
        k = done.value
        return IterResult(w, wl2, None, self.deltas[:k], k)


def rank_csr_sharded(n: int, starts, row_ptr_local, col_idx_local, cap, bg, b0, max_iters: int = 200,
                     tol: float = 1e-7, want_l2: bool = True, group=None, check_every: int = 8, lib=None,
                     all_gather=None):
    """MAPI ranking (Eq. 13) with the destination rows partitioned over the ranks:
    rank r holds the sub-CSR of rows [starts[r], starts[r+1]) (csr_row_partition / csr_shard) and the full
    cap / bg / b0.  Per iteration: the local gather, ONE collective (the all-gather of the e_t blocks, in
    place in the workspace, n * 4 bytes in total) and the node kernels on the full state, which every rank
    runs identically — no all-reduce of s_t or delta_t is needed and all ranks take the same stop decision.
    With tol > 0 the host reads the device stop flag every `check_every` iterations (the launches enqueued
    after a stop return at once on the device).  all_gather(e_full, starts, rank) is injectable."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if len(starts) != world + 1 or starts[0] != 0 or starts[-1] != n:
        raise ValueError(f"starts must have world + 1 = {world + 1} entries from 0 to n")
    r0, r1 = int(starts[rank]), int(starts[rank + 1])
    if int(row_ptr_local.numel()) - 1 != r1 - r0:
        raise ValueError(f"row_ptr_local has {int(row_ptr_local.numel()) - 1} rows; the partition gives {r1 - r0}")
    ses = CsrShardSession(n, r0, row_ptr_local, col_idx_local, cap, bg, b0, max_iters, tol, lib=lib)
    if all_gather is None:
        all_gather = _e_all_gather(group, world)
    ses.begin()
    for t in range(max_iters):
        ses.rows(t)
        if world > 1:
            all_gather(ses.e_view(t), starts, rank)
        ses.normalize(t)
        if tol > 0.0 and (t + 1) % max(1, check_every) == 0 and t + 1 < max_iters:
            if ses.poll()[1]:
                break
    return ses.finish(want_l2)


def _e_all_gather(group, world):
    """In-place all-gather of the ranks' row blocks of e_t: one NCCL all-gather when the blocks are equal,
    else one broadcast per non-empty block (NCCL groups uneven all-gathers the same way)."""
    import torch.distributed as dist

    def gather(e_full, starts, rank):
        sizes = [starts[q + 1] - starts[q] for q in range(world)]
        if len(set(sizes)) == 1:
            dist.all_gather_into_tensor(e_full, e_full[starts[rank]:starts[rank + 1]].clone(), group=group)
            return
        for q in range(world):
            if sizes[q]:
                dist.broadcast(e_full[starts[q]:starts[q + 1]], src=dist.get_global_rank(group, q) if group else q,
                               group=group)

    return gather
