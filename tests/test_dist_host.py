"""N > 1 host logic on CPU (gloo, world_size 2): the bench's max-over-ranks timing and the
reference arm's rank-0-only rule (replicas, no data-path collective)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    import torch.distributed as tdist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    t = bench.max_over_ranks(10.0 + 5.0 * rank)  # rank 1 is the slow one

    class Args:  # the reference arm returns nothing on ranks != 0
        workload = "cfg1"
        steps = 1
        warmup = 0

    ref = bench.run_reference(Args, rank, world) if rank != 0 else "skipped"
    q.put((rank, t, ref))
    tdist.barrier()
    tdist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = {r: (t, ref) for r, t, ref in out}
    assert got[0][0] == 15.0 and got[1][0] == 15.0  # every rank sees the max
    assert got[1][1] is None  # only rank 0 runs the reference arm


def test_max_over_ranks_single_process():
    import bench

    assert bench.max_over_ranks(3.5) == 3.5


# ---------------------------------------------------------------- row-sharded MAPI orchestration (NEXT-4)


def _sharded_worker(rank, world, port, q):
    import sys

    import numpy as np
    import torch
    import torch.distributed as tdist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2110_12065_b200.sharded import iterate_sharded, row_partition

    n = 48
    r = np.random.default_rng(3)
    A = (r.standard_normal((n, n)) + np.eye(n) * 2).astype(np.float32)
    b0 = np.full(n, 1 / np.sqrt(n), np.float32)
    r0, r1 = row_partition(n, world, rank)

    # CPU stand-ins for the CUDA steps (test only): oracle mat-vec of the local rows, and the
    # Algorithm 1 normalisation written out in numpy (fp64, fixed order)
    def local_matvec(A_loc, w, y_loc):
        y_loc.copy_(torch.from_numpy(oracle.matvec(A_loc.numpy(), w.numpy().astype(np.float64)).astype(np.float32)))

    def normalize(y, w, s_out, d_out, st_out):
        yv = y.numpy().astype(np.float64)
        s = np.sum(np.abs(yv))
        wn = (yv / s).astype(np.float32)
        d_out[0] = float(np.sum(np.abs(wn.astype(np.float64) - w.numpy().astype(np.float64))))
        s_out[0] = s
        st_out[0] = 0
        w.copy_(torch.from_numpy(wn))

    res = iterate_sharded(torch.from_numpy(A[r0:r1].copy()), n, torch.from_numpy(b0), 12,
                          local_matvec=local_matvec, normalize=normalize,
                          all_gather=lambda full, part: tdist.all_gather_into_tensor(full, part))
    q.put((rank, res.w.numpy().copy(), res.norms.numpy().copy(), res.iters_done))
    tdist.barrier()
    tdist.destroy_process_group()


def test_row_sharded_mapi_gloo_world2():
    """Two ranks, each holding half of A's rows: every rank ends with the same w, equal to the
    single-process MAPI of the oracle (the shard/gather/normalise orchestration of DESIGN.md §8)."""
    import numpy as np

    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {r: (w, nr, k) for r, w, nr, k in [q.get(timeout=180) for _ in range(2)]}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(out[0][0], out[1][0])  # identical on every rank
    n = 48
    r = np.random.default_rng(3)
    A = (r.standard_normal((n, n)) + np.eye(n) * 2).astype(np.float32)
    ref = oracle.mapi(A, np.full(n, 1 / np.sqrt(n), np.float32), 12)
    np.testing.assert_allclose(out[0][0], ref.w, rtol=2e-6, atol=1e-7)
    np.testing.assert_allclose(out[0][1], ref.norms, rtol=1e-6)
    assert out[0][2] == 12


def _batched_worker(rank, world, port, q):
    import sys

    import numpy as np
    import torch
    import torch.distributed as tdist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2110_12065_b200 import BatchedResult
    from paper_2110_12065_b200.sharded import iterate_batched_sharded

    n, k, T = 40, 6, 9
    r = np.random.default_rng(5)
    A = (r.standard_normal((n, n)) + 2 * np.eye(n)).astype(np.float32)
    B0 = r.standard_normal((k, n)).astype(np.float32)
    B0 /= np.linalg.norm(B0, axis=1, keepdims=True)

    def run_local(A_, B_, iters, tol, op):  # CPU stand-in for mapi_iterate_batched (test only): the oracle per vector
        rs = [oracle.mapi(A_.numpy(), b.numpy(), iters) for b in B_]
        return BatchedResult(torch.from_numpy(np.stack([x.w for x in rs]).astype(np.float32)),
                             torch.from_numpy(np.stack([x.norms for x in rs], 1).astype(np.float32)), None,
                             [x.iters_done for x in rs])

    k0, k1, (W, norms, done) = iterate_batched_sharded(torch.from_numpy(A), torch.from_numpy(B0), T, run_local=run_local,
                                                       gather=True)
    q.put((rank, k0, k1, W.numpy().copy(), norms.numpy().copy(), done.numpy().copy()))
    tdist.barrier()
    tdist.destroy_process_group()


def test_batched_k_sharded_gloo_world2():
    """cfg4's k independent runs split over two ranks (no data-path collective): the slices tile [0, k), and the
    gathered W / norms equal the oracle's per-vector MAPI in the single-GPU (vector-major) layout."""
    import numpy as np

    import oracle
    from paper_2110_12065_b200.sharded import vector_partition

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batched_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {r: rest for r, *rest in [q.get(timeout=180) for _ in range(2)]}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert (out[0][0], out[0][1], out[1][0], out[1][1]) == (0, 3, 3, 6)
    np.testing.assert_array_equal(out[0][2], out[1][2])
    n, k, T = 40, 6, 9
    r = np.random.default_rng(5)
    A = (r.standard_normal((n, n)) + 2 * np.eye(n)).astype(np.float32)
    B0 = r.standard_normal((k, n)).astype(np.float32)
    B0 /= np.linalg.norm(B0, axis=1, keepdims=True)
    for j in range(k):
        ref = oracle.mapi(A, B0[j], T)
        np.testing.assert_allclose(out[0][2][j], ref.w, rtol=2e-6, atol=1e-7)
        np.testing.assert_allclose(out[0][3][:, j], ref.norms, rtol=1e-6)
    assert list(out[0][4]) == [T] * k
    for world in (1, 2, 3, 5, 8):  # the slices tile [0, k) for any world, k not divisible included
        cuts = [vector_partition(7, world, rr) for rr in range(world)]
        assert cuts[0][0] == 0 and cuts[-1][1] == 7 and all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))


def test_row_partition():
    from paper_2110_12065_b200.sharded import row_partition

    assert [row_partition(32768, 8, r) for r in (0, 7)] == [(0, 4096), (28672, 32768)]
    import pytest

    with pytest.raises(ValueError):
        row_partition(10, 3, 0)


# ---------------------------------------------------------------- fused P2P exchange set-up (K2p)


class _FakeP2PLib:
    """Stand-in for libmapi's six exchange entry points (host logic only): addresses encode ranks."""

    def __init__(self, rank):
        self.rank = rank
        self.closed, self.freed = [], []

    def mapi_p2p_exchange_bytes(self, n, world):
        return 256 + 8 * n + 16 * world

    def mapi_p2p_alloc(self, nbytes, ptr_ref):
        ptr_ref._obj.value = 0x100000 * (self.rank + 1)
        return 0

    def mapi_ipc_get_handle(self, ptr, handle):
        handle.raw = bytes([self.rank + 1]) * 64
        return 0

    def mapi_ipc_open_handle(self, handle, ptr_ref):
        ptr_ref._obj.value = 0xA0000000 + handle.raw[0]
        return 0

    def mapi_ipc_close_handle(self, ptr):
        self.closed.append(ptr)
        return 0

    def mapi_p2p_free(self, ptr):
        self.freed.append(ptr)
        return 0

    def mapi_last_error_message(self):
        return b""


def _p2p_setup_worker(rank, world, port, q):
    import sys

    import torch.distributed as tdist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2110_12065_b200.sharded import P2PExchange

    def allgather(b):
        out = [None] * world
        tdist.all_gather_object(out, b)
        return out

    lib = _FakeP2PLib(rank)
    ex = P2PExchange(96, rank, world, lib=lib, allgather=allgather, sms=148 - 4 * rank)
    peers = list(ex.peer_addrs)
    ex.advance(7)
    ex.advance(3)
    adv = (ex.epoch, ex.flag_base, ex.grid)
    ex.close()
    q.put((rank, peers, adv, sorted(lib.closed), lib.freed))
    tdist.barrier()
    tdist.destroy_process_group()


def test_p2p_exchange_setup_gloo_world3():
    """K2p / K2sp host set-up with three ranks: IPC handles all-gathered in rank order, peers[rank] is the
    own buffer and peers[q] the mapping of rank q's handle, every rank agrees on the same grid (the minimum
    SM count), the epoch / flag base advance by the published iterations (x world: one arrival per rank per
    iteration), and close() unmaps every peer and frees the own buffer."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    procs = [ctx.Process(target=_p2p_setup_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {r: rest for r, *rest in [q.get(timeout=180) for _ in range(world)]}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        peers, adv, closed, freed = out[r]
        own = 0x100000 * (r + 1)
        assert peers == [own if p == r else 0xA0000000 + p + 1 for p in range(world)]
        assert adv == (10, 10 * world, 148 - 4 * (world - 1))
        assert closed == sorted(0xA0000000 + p + 1 for p in range(world) if p != r)
        assert freed == [own]


# ------------------------------------------------- sharded symmetric K2sp: the task / row partition on CPU


def _sym_lib():
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2110_12065_b200 as m

    m.build()
    return m.load()


def _task_start(b, nc):  # sum_{b' < b} (nc - b' // 2): an independent restatement of the task numbering
    return sum(nc - bb // 2 for bb in range(b))


def _valid(lib, n, rank, world, j):
    import ctypes

    out = (ctypes.c_int64 * 4)()
    assert lib.mapi_sym_shard_valid(n, rank, world, j, out) == 0
    return tuple(out)


def test_sym_shard_partition():
    """K2sp's split of K2s's upper-triangle task list (mapi_sym_shard_rows / mapi_sym_shard_valid, host-only
    C): the ranks' task ranges tile [0, T); each rank's held rows contain every strip its tasks read; and for
    every row j the ranks' valid row-partial chunks and column-partial blocks are disjoint, cover
    [c(j), nc) and [0, b(j)], and are exactly the partials of the tasks the rank owns (checked against an
    independent enumeration of the task indices)."""
    from paper_2110_12065_b200.sharded import sym_shard

    lib = _sym_lib()
    RB, CC = 128, 256
    for n in (8, 1000, 8192, 33000):
        nb, nc = -(-n // RB), -(-n // CC)
        T = _task_start(nb, nc)
        for world in (1, 2, 3, 8):
            shards = [sym_shard(n, r, world, lib) for r in range(world)]
            assert shards[0][2] == 0 and shards[-1][3] == T
            for r in range(world - 1):
                assert shards[r][3] == shards[r + 1][2]
            starts = [_task_start(b, nc) for b in range(nb + 1)]
            owner = {}
            for r, (lo, hi, tlo, thi) in enumerate(shards):
                for b in range(nb):
                    for c in range(b // 2, nc):
                        t = starts[b] + c - b // 2
                        if tlo <= t < thi:
                            owner[(b, c)] = r
                            assert lo <= b * RB and min(n, (b + 1) * RB) <= hi, (n, world, r, b)
            rows = range(n) if n <= 1000 else list(range(0, n, 97)) + [n - 1]
            for j in rows:
                B, C = j // RB, j // CC
                got = [_valid(lib, n, r, world, j) for r in range(world)]
                for r, (clo, chi, blo, bhi) in enumerate(got):
                    mine_c = {c for c in range(C, nc) if owner[(B, c)] == r}
                    mine_b = {b for b in range(B + 1) if owner[(b, C)] == r}
                    assert set(range(clo, chi)) == mine_c, (n, world, r, j)
                    assert set(range(blo, bhi)) == mine_b, (n, world, r, j)


def _sym_sharded_worker(rank, world, port, q):
    import sys

    import numpy as np
    import torch
    import torch.distributed as tdist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    lib = _sym_lib()
    n, RB, CC = 1000, 128, 256
    r = np.random.default_rng(21)
    G = r.standard_normal((n, n))
    A = np.triu(G) + np.triu(G, 1).T
    w = r.standard_normal(n)

    def term(a, x):  # MAVP term, Eq. (3): sign(a x) min(|a|, |x|)
        return np.sign(a * x) * np.minimum(np.abs(a), np.abs(x))

    # this rank's partial y from the partials its tasks produce (row terms k >= j of its chunks, column terms
    # k < j of its row blocks), reading only the upper triangle
    y = np.zeros(n)
    for j in range(n):
        clo, chi, blo, bhi = _valid(lib, n, rank, world, j)
        for c in range(clo, chi):
            k = np.arange(max(j, c * CC), min(n, (c + 1) * CC))
            y[j] += term(A[j, k], w[k]).sum()
        for b in range(blo, bhi):
            k = np.arange(b * RB, min(j, (b + 1) * RB))
            y[j] += term(A[k, j], w[k]).sum()
    t = torch.from_numpy(y)
    tdist.all_reduce(t)  # the exchange step: the sum of the ranks' partial y vectors
    q.put((rank, t.numpy().copy()))
    tdist.barrier()
    tdist.destroy_process_group()


def test_sym_sharded_partials_gloo_world3():
    """Three ranks each compute the partial y of their slice of the upper-triangle task list (the valid
    ranges of mapi_sym_shard_valid); after the exchange (a sum over the ranks) every rank holds y = A (+) w of
    the full symmetric matrix (oracle mat-vec), i.e. every MAVP term is produced by exactly one rank."""
    import numpy as np

    import oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    procs = [ctx.Process(target=_sym_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 1000
    r = np.random.default_rng(21)
    G = r.standard_normal((n, n))
    A = np.triu(G) + np.triu(G, 1).T
    w = r.standard_normal(n)
    ref = oracle.matvec(A, w)
    for k in range(world):
        np.testing.assert_array_equal(out[k], out[0])
    np.testing.assert_allclose(out[0], ref, rtol=1e-12, atol=1e-9)


# -------------------------------------------------------- CSR ranking over ranks (K3n): orchestration on CPU


class _FakeCsrShardLib:
    """Stand-in for mapi_rank_csr_shard_* (host orchestration test only; test code, so it may restate the
    exact sparse + background form of Eq. 13 in numpy fp64): the pointers are those of CPU tensors, e_t lives
    in the caller's workspace at the library's offsets so that the in-place collective works on it."""

    def __init__(self):
        self.state = {}

    @staticmethod
    def _arr(ptr, count, dtype):
        import ctypes

        import numpy as np

        if count == 0:
            return np.zeros(0, dtype)
        size = count * np.dtype(dtype).itemsize
        return np.frombuffer((ctypes.c_char * size).from_address(ptr), dtype=dtype)

    def mapi_workspace_size(self, op, n, nnz, k):
        return 256 + 2 * ((4 * n + 255) & ~255)

    def _e(self, ws, n, t):
        import numpy as np

        return self._arr(ws + 256 + (t & 1) * ((4 * n + 255) & ~255), n, np.float32)

    def mapi_rank_csr_shard_begin(self, n, m, nnz, rp, cap, bg, b0, ws, need, sp):
        import numpy as np

        f = np.float32
        self.state[ws] = dict(w=self._arr(b0, n, f).astype(np.float64), cap=self._arr(cap, n, f).astype(np.float64),
                              bg=self._arr(bg, n, f).astype(np.float64), done=0, stop=0)
        return 0

    def mapi_rank_csr_shard_rows(self, n, m, row0, nnz, rp, ci, t, e_out, ws, need, sp):
        import numpy as np

        s = self.state[ws]
        if e_out is not None:
            e_out._obj.value = ws + 256 + (t & 1) * ((4 * n + 255) & ~255)
        if s["stop"]:
            return 0
        v = np.minimum(np.maximum(s["w"] - s["bg"], 0.0), s["cap"])
        rp_ = self._arr(rp, m + 1, np.int32)
        ci_ = self._arr(ci, nnz, np.int32) if nnz else np.zeros(0, np.int32)
        e = self._e(ws, n, t)
        for i in range(m):
            e[row0 + i] = v[ci_[rp_[i]:rp_[i + 1]]].sum()
        return 0

    def mapi_rank_csr_shard_normalize(self, n, m, nnz, cap, bg, b0, t, tol, deltas, ws, need, sp):
        import numpy as np

        s = self.state[ws]
        if s["stop"]:
            return 0
        S = np.minimum(s["bg"], s["w"]).sum()
        y = S + self._e(ws, n, t).astype(np.float64)
        wn = y / y.sum()
        d = np.abs(wn - s["w"]).sum()
        self._arr(deltas, t + 1, np.float32)[t] = d
        s["w"], s["done"] = wn, t + 1
        if tol > 0 and d < tol:
            s["stop"] = 1
        return 0

    def mapi_rank_csr_shard_finish(self, n, m, nnz, b0, w_out, w_l2, done, stopped, ws, need, sp):
        import numpy as np

        s = self.state[ws]
        if w_out:
            self._arr(w_out, n, np.float32)[:] = s["w"]
            if w_l2:
                self._arr(w_l2, n, np.float32)[:] = s["w"] / np.linalg.norm(s["w"])
        if done is not None:
            done._obj.value = s["done"]
        if stopped is not None:
            stopped._obj.value = s["stop"]
        return 0

    def mapi_last_error_message(self):
        return b""


def _csr_sharded_worker(rank, world, port, q):
    import sys

    import numpy as np
    import torch
    import torch.distributed as tdist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_2110_12065_b200.sharded import csr_row_partition, csr_shard, rank_csr_sharded

    n = 257
    edges, row_ptr, col_idx = synth.random_graph(n, 0.04, seed=11, n_dangling=25)
    outdeg = np.bincount(edges[:, 0], minlength=n)
    alpha = 0.85
    with np.errstate(divide="ignore"):
        cap = np.where(outdeg > 0, alpha / outdeg, 0.0).astype(np.float32)
    bg = np.where(outdeg > 0, (1 - alpha) / n, 1.0 / n).astype(np.float32)
    starts = csr_row_partition(row_ptr, world)
    rp = torch.from_numpy(row_ptr.astype(np.int32))
    ci = torch.from_numpy(col_idx.astype(np.int32))
    rpl, cil = csr_shard(rp, ci, starts[rank], starts[rank + 1])
    b0 = torch.full((n,), 1.0 / n, dtype=torch.float32)
    out = {}
    for name, tol, iters in (("fixed", 0.0, 12), ("tol", 1e-7, 200)):
        res = rank_csr_sharded(n, starts, rpl, cil, torch.from_numpy(cap), torch.from_numpy(bg), b0, iters, tol,
                               lib=_FakeCsrShardLib(), check_every=3)
        out[name] = (res.w.numpy().copy(), res.deltas.numpy().copy(), res.iters_done)
    q.put((rank, starts, out))
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_csr_rank_sharded_gloo(world):
    """sharded.rank_csr_sharded over gloo: the row partition tiles [0, n) with balanced rows + in-edges, the
    in-place exchange of the e_t blocks (uneven blocks: one broadcast per owner) delivers every owner's rows
    to every rank, all ranks finish with the same w / deltas / iteration count (fixed count and tol stop with
    a periodic host check), and the result is the oracle's rank_csr."""
    import numpy as np

    import oracle
    import synth

    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_csr_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {r: rest for r, *rest in [q.get(timeout=180) for _ in range(world)]}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 257
    edges, row_ptr, col_idx = synth.random_graph(n, 0.04, seed=11, n_dangling=25)
    b0 = np.full(n, 1.0 / n, dtype=np.float32)
    starts = got[0][0]
    assert starts[0] == 0 and starts[-1] == n and all(a <= b for a, b in zip(starts, starts[1:]))
    items = [(starts[r + 1] - starts[r]) + int(row_ptr[starts[r + 1]] - row_ptr[starts[r]]) for r in range(world)]
    assert max(items) - min(items) <= 2 * (1 + int(np.max(np.diff(row_ptr))))
    for name, tol, iters in (("fixed", 0.0, 12), ("tol", 1e-7, 200)):
        ref = oracle.rank_csr(n, row_ptr, col_idx, b0=b0, max_iters=iters, tol=tol)
        w0, d0, k0 = got[0][1][name]
        for r in range(1, world):
            w, d, k = got[r][1][name]
            assert k == k0 and np.array_equal(w, w0) and np.array_equal(d, d0)
        assert k0 == ref.iters_done
        np.testing.assert_allclose(w0, ref.w, rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(d0, ref.deltas, rtol=1e-3, atol=1e-9)
