"""GPU parity of the dense MAVP mat-vec (K1) and the MAPI iteration (K2) against the fp64 oracle.

Tolerances (from the BASELINE north star):
  T1 single mat-vec:  |y_gpu_j - y_orc_j| <= 1e-5 * mag_j,  mag_j = sum_k |term_jk|
  T2 after T iterations, on the l2-normalised vectors: |cos| >= 1 - 1e-6 and max|diff| <= 1e-4;
     per-iteration norms s_t relative <= 1e-5.
All calls go through the C ABI (paper_2110_12065_b200 -> libmapi.so).
"""
import os

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

T1 = 1e-5


def _t1(y_gpu, y_orc, mag):
    y_gpu = np.asarray(y_gpu, np.float64)
    err = np.abs(y_gpu - y_orc)
    bound = T1 * mag
    bad = np.nonzero(err > bound)[0]
    assert bad.size == 0, (f"T1 violated at {bad[:5]}: err {err[bad[:5]]}, bound {bound[bad[:5]]}, "
                           f"y_gpu {y_gpu[bad[:5]]}, y_orc {y_orc[bad[:5]]}")


def _t2(w_gpu_l2, w_orc, norms_gpu=None, norms_orc=None):
    a = np.asarray(w_gpu_l2, np.float64)
    b = np.asarray(w_orc, np.float64)
    b = b / np.linalg.norm(b)
    cos = float(a @ b / np.linalg.norm(a))
    assert abs(cos) >= 1 - 1e-6, f"|cos| = {abs(cos)!r}"
    assert np.max(np.abs(a - b)) <= 1e-4, f"max abs diff {np.max(np.abs(a - b))}"
    if norms_gpu is not None:
        ng = np.asarray(norms_gpu, np.float64)
        np.testing.assert_allclose(ng, norms_orc, rtol=1e-5)


SHAPES = [(1, 1), (1, 7), (3, 5), (9, 9), (31, 33), (33, 31), (255, 256), (256, 257), (257, 255),
          (100, 4109), (64, 32768), (7, 70001)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("pad", [0, 1, 4, 8])
def test_matvec_t1(mapi_lib, orc, shape, pad):
    m = mapi_lib
    n_rows, n_cols = shape
    for op, opname in ((m.MIN1, "min1"), (m.MIN2, "min2")):
        for kind in ("normal", "mixed"):
            seed = hash((n_rows, n_cols, pad, op, kind)) % (2 ** 31)
            M, lda = synth.random_matrix(n_rows, n_cols, seed=seed, lda=n_cols + pad, kind=kind)
            x = synth.random_vector(n_cols, seed=seed + 1, kind="mixed" if kind == "mixed" else "normal")
            Ad = torch.from_numpy(M).cuda()
            y = m.mavp_matvec(Ad[:, :n_cols], torch.from_numpy(x).cuda(), op=op)
            torch.cuda.synchronize()
            y_orc, mag = orc.matvec(M[:, :n_cols], x, opname, return_mag=True)
            _t1(y.cpu().numpy(), y_orc, mag)


def test_matvec_spec_examples_exact(mapi_lib):
    m = mapi_lib
    A = torch.tensor([[1.0, 0.0], [0.0, 1.0]], device="cuda")
    y = m.mavp_matvec(A, torch.tensor([5.0, -7.0], device="cuda"))
    assert y.tolist() == [1.0, -1.0]
    y = m.mavp_matvec(torch.tensor([[2.0, 2.0]], device="cuda"), torch.zeros(2, device="cuda"))
    assert y.tolist() == [0.0]
    x = torch.tensor([1.0, -2.0, 3.0], device="cuda")
    assert m.mavp_matvec(x[None, :], x).tolist() == [6.0]  # l1 induction
    y = m.mavp_matvec(torch.tensor([[1.0]], device="cuda"), torch.tensor([-1.0], device="cuda"), op=m.MIN2)
    assert y.tolist() == [0.0]


def test_matvec_degenerate_shapes(mapi_lib):
    m = mapi_lib
    A = torch.empty(5, 0, device="cuda")
    y = torch.full((5,), 3.0, device="cuda")
    m.mavp_matvec(A, torch.empty(0, device="cuda"), y)
    torch.cuda.synchronize()
    assert y.tolist() == [0.0] * 5
    m.mavp_matvec(torch.empty(0, 4, device="cuda"), torch.ones(4, device="cuda"), torch.empty(0, device="cuda"))


def test_matvec_bitwise_oddness_and_symmetry(mapi_lib):
    m = mapi_lib
    M, _ = synth.random_matrix(300, 1000, seed=5)
    x = synth.random_vector(1000, seed=6)
    A = torch.from_numpy(M).cuda()
    xd = torch.from_numpy(x).cuda()
    y1 = m.mavp_matvec(A, xd)
    y2 = m.mavp_matvec(A, -xd)
    assert torch.equal(y1, -y2)  # (-x) (+) a = -(x (+) a), bitwise
    # symmetry x (+) a = a (+) x: row j against x vs x (as a 1-row matrix) against row j
    j = 17
    ya = m.mavp_matvec(xd[None, :].contiguous(), A[j].contiguous())
    assert torch.equal(ya[0], y1[j])


# ------------------------------------------------------------------------------ iteration


def _iterate_case(m, orc, A32, b0, iters, tol=0.0, op="min1"):
    res = m.iterate(torch.from_numpy(A32).cuda(), torch.from_numpy(b0).cuda(), iters, tol,
                    op=m.MIN1 if op == "min1" else m.MIN2)
    ref = orc.mapi(A32, b0.astype(np.float64), iters, tol, op=op)
    return res, ref


def test_iterate_cfg1_parity(mapi_lib, orc):
    cfg = synth.cfg1()
    res, ref = _iterate_case(mapi_lib, orc, cfg["A"], cfg["b0"], cfg["iters"])
    assert res.iters_done == ref.iters_done == 50
    _t2(res.w_l2.cpu().numpy(), ref.w, res.norms.cpu().numpy(), ref.norms)
    np.testing.assert_allclose(res.deltas.cpu().numpy(), ref.deltas, rtol=1e-3, atol=1e-7)
    np.testing.assert_allclose(res.w.cpu().numpy(), ref.w, atol=1e-6)
    assert abs(float(res.w.abs().sum()) - 1.0) < 1e-5


@pytest.mark.parametrize("n", [1, 2, 7, 33, 255, 1000, 4099])
@pytest.mark.parametrize("op", ["min1", "min2"])
def test_iterate_random_nonsymmetric(mapi_lib, orc, n, op):
    r = np.random.default_rng(n)
    A = r.standard_normal((n, n)).astype(np.float32)
    if op == "min2":
        A = np.abs(A) + np.eye(n, dtype=np.float32)
    b0 = (np.abs(r.standard_normal(n)) + 0.1).astype(np.float32)
    b0 /= np.linalg.norm(b0)
    res, ref = _iterate_case(mapi_lib, orc, A, b0, 25, op=op)
    assert res.iters_done == ref.iters_done
    _t2(res.w_l2.cpu().numpy(), ref.w, res.norms.cpu().numpy(), ref.norms)


def test_iterate_padded_lda_and_unaligned(mapi_lib, orc):
    m = mapi_lib
    for pad in (1, 3, 4, 8):
        M, lda = synth.random_matrix(300, 300, seed=pad, lda=300 + pad)
        M[:, :300] += np.eye(300, dtype=np.float32) * 5
        b0 = np.full(300, 1 / np.sqrt(300), np.float32)
        Ad = torch.from_numpy(M).cuda()[:, :300]
        res = m.iterate(Ad, torch.from_numpy(b0).cuda(), 20)
        ref = orc.mapi(np.ascontiguousarray(M[:, :300]), b0, 20)
        _t2(res.w_l2.cpu().numpy(), ref.w, res.norms.cpu().numpy(), ref.norms)


def test_iterate_tolerance_stop_and_identity(mapi_lib, orc):
    m = mapi_lib
    n = 64
    A = np.eye(n, dtype=np.float32)
    b0 = np.linspace(0.1, 1.0, n).astype(np.float32)
    b0 /= np.linalg.norm(b0)
    res = m.iterate(torch.from_numpy(A).cuda(), torch.from_numpy(b0).cuda(), 50, tol=1e-6)
    ref = orc.mapi(A, b0, 50, tol=1e-6)
    assert res.iters_done == ref.iters_done == 2  # A = I: fixed point after one step
    np.testing.assert_allclose(res.w.cpu().numpy(), b0 / np.abs(b0).sum(), rtol=2e-7)


def test_iterate_degenerate(mapi_lib):
    m = mapi_lib
    A = torch.zeros(40, 40, device="cuda")
    b0 = torch.full((40,), 0.1, device="cuda")
    with pytest.raises(m.MapiError) as ei:
        m.iterate(A, b0, 10)
    assert ei.value.name == "MAPI_ERR_DEGENERATE" and ei.value.iters_done == 0


def test_iterate_determinism_equivariance_resume(mapi_lib):
    m = mapi_lib
    cfg = synth.cfg1()
    A = torch.from_numpy(cfg["A"]).cuda()
    b0 = torch.from_numpy(cfg["b0"]).cuda()
    r1 = m.iterate(A, b0, 30)
    r2 = m.iterate(A, b0, 30)
    assert torch.equal(r1.w, r2.w) and torch.equal(r1.norms, r2.norms) and torch.equal(r1.deltas, r2.deltas)
    rn = m.iterate(A, -b0, 30)
    assert torch.equal(rn.w, -r1.w)  # sign equivariance, bitwise
    a = m.iterate(A, b0, 12)
    b = m.iterate(A, a.w.clone(), 18)
    assert torch.equal(b.w, r1.w)  # resume == uninterrupted run (checkpoint state is (w_t, t))
    assert torch.equal(b.norms, r1.norms[12:])


def test_iterate_multilaunch_path_matches(mapi_lib, orc, monkeypatch):
    m = mapi_lib
    cfg = synth.cfg1()
    monkeypatch.setenv("MAPI_DENSE_PATH", "multi")
    res = m.iterate(torch.from_numpy(cfg["A"]).cuda(), torch.from_numpy(cfg["b0"]).cuda(), 50)
    ref = orc.mapi(cfg["A"], cfg["b0"], 50)
    _t2(res.w_l2.cpu().numpy(), ref.w, res.norms.cpu().numpy(), ref.norms)


def test_iterate_host_buffers(mapi_lib, orc):
    m = mapi_lib
    cfg = synth.cfg1()
    A = torch.from_numpy(cfg["A"]).pin_memory()
    b0 = torch.from_numpy(cfg["b0"]).pin_memory()
    res = m.iterate_host(A, b0, 50)
    dev = m.iterate(A.cuda(), b0.cuda(), 50)
    assert torch.equal(res.w, dev.w.cpu()) and torch.equal(res.norms, dev.norms.cpu())


# ------------------------------------------------------------------------------ full size (cfg3)


@pytest.fixture(scope="module")
def cfg3_device():
    cfg = synth.cfg3(device="cuda")
    return cfg


@pytest.fixture(scope="module")
def cfg3_oracle(orc, cfg3_device):
    """The fp64 oracle's 100 MAPI iterations (Alg. 1) on the fp32 bytes of cfg3's A: ~1 min on
    the box's host cores.  Shared by the end-to-end tests of both kernels."""
    A_host = cfg3_device["A"].cpu().numpy()
    ref = orc.mapi(A_host, cfg3_device["b0"].astype(np.float64), cfg3_device["iters"])
    assert ref.status == orc.OK and ref.iters_done == 100
    return ref


@pytest.mark.parametrize("kernel", ["sym", "full"])
def test_cfg3_end_to_end_vs_oracle(mapi_lib, cfg3_oracle, cfg3_device, kernel):
    """The headline workload exactly as bench.py times it (BASELINE configs[2]: 32768^2, 100 iterations,
    b0 = 1/sqrt(n)) against the fp64 oracle's own 100-iteration trajectory (no conditioning on the GPU's
    iterates): T2 on the final l2 vector (|cos| >= 1 - 1e-6, max|diff| <= 1e-4), every per-iteration norm
    s_t within 1e-5 relative, the l1 iterate within 1e-6 absolute.  kernel = "sym" is mapi_iterate_sym (K2s,
    the bench path, upper triangle only); "full" is mapi_iterate (K2c, all n^2 entries)."""
    m = mapi_lib
    A = cfg3_device["A"]
    b0 = torch.from_numpy(cfg3_device["b0"]).cuda()
    res = (m.iterate_sym if kernel == "sym" else m.iterate)(A, b0, 100)
    assert res.iters_done == 100
    _t2(res.w_l2.cpu().numpy(), cfg3_oracle.w, res.norms.cpu().numpy(), cfg3_oracle.norms)
    np.testing.assert_allclose(res.w.cpu().numpy(), cfg3_oracle.w, rtol=0, atol=1e-6)
    np.testing.assert_allclose(res.deltas.cpu().numpy(), cfg3_oracle.deltas, rtol=1e-3)


def test_cfg3_matvec_sampled_rows(mapi_lib, orc, cfg3_device):
    """Full BASELINE size (32768^2, 4 GiB) in the bench launch configuration: T1 on 512 sampled
    rows of one mat-vec from the b0 start and from a rough iterate."""
    m = mapi_lib
    A = cfg3_device["A"]
    n = A.shape[0]
    r = np.random.default_rng(0)
    rows = np.sort(r.choice(n, 512, replace=False))
    A_rows = A[torch.from_numpy(rows).cuda()].cpu().numpy()
    for x in (cfg3_device["b0"], (r.standard_normal(n) / n).astype(np.float32)):
        y = m.mavp_matvec(A, torch.from_numpy(x).cuda()).cpu().numpy()
        y_orc, mag = orc.matvec(A_rows, x, return_mag=True)
        _t1(y[rows], y_orc, mag)


def test_cfg3_last_step_and_invariants(mapi_lib, orc, cfg3_device):
    """cfg3 as bench.py runs it (100 iterations, persistent kernel): the GPU's 100th iterate must
    equal the oracle's fp64 step applied to the GPU's own 99th iterate (per-element T1-scaled bound),
    s_99 must match, ||w||_1 = 1, and the run is bitwise reproducible."""
    m = mapi_lib
    A = cfg3_device["A"]
    b0 = torch.from_numpy(cfg3_device["b0"]).cuda()
    r100 = m.iterate(A, b0, 100)
    r99 = m.iterate(A, b0, 99)
    assert torch.equal(r100.norms[:99], r99.norms)
    w99 = r99.w.cpu().numpy()
    A_host = A.cpu().numpy()
    y, mag = orc.matvec(A_host, w99, return_mag=True)
    s = np.abs(y).sum()
    assert abs(float(r100.norms[99]) - s) <= 1e-5 * s
    w100 = r100.w.cpu().numpy().astype(np.float64)
    err = np.abs(w100 - y / s)
    assert np.all(err <= 1e-5 * mag / s + 2e-5 * np.abs(y / s)), float(np.max(err))
    assert abs(np.abs(w100).sum() - 1.0) < 1e-5
    r100b = m.iterate(A, b0, 100)
    assert torch.equal(r100.w, r100b.w)


@pytest.mark.parametrize("path", ["single", "cluster", "cluster_smem", "rows", "coop", "bulk", "resident", "multi"])
@pytest.mark.parametrize("n", [256, 511, 4096, 8200])
def test_every_dense_path_matches_oracle(mapi_lib, orc, monkeypatch, path, n):
    """Each dense iteration kernel (K6 cluster, K2 per-row, K2c cooperative rows, multi-launch),
    forced through MAPI_DENSE_PATH, against the oracle (T2).  Paths a shape cannot use fall back."""
    m = mapi_lib
    r = np.random.default_rng(n)
    A = r.standard_normal((n, n)).astype(np.float32)
    A += np.diag(np.abs(r.standard_normal(n)) * 4).astype(np.float32)
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    monkeypatch.setenv("MAPI_DENSE_PATH", path)
    res = m.iterate(torch.from_numpy(A).cuda(), torch.from_numpy(b0).cuda(), 20)
    ref = orc.mapi(A, b0, 20)
    assert res.iters_done == 20
    _t2(res.w_l2.cpu().numpy(), ref.w, res.norms.cpu().numpy(), ref.norms)


@pytest.mark.parametrize("n,pad", [(1024, 0), (1500, 4), (2052, 8), (4096, 0), (5000, 12)])
@pytest.mark.parametrize("op", ["min1", "min2"])
def test_bulk_ring_path(mapi_lib, orc, monkeypatch, n, pad, op):
    """K2t (TMA bulk-copy ring): ragged last chunk (n % 1024 != 0), padded lda, both MAVP operators,
    vs the oracle (T2), bitwise reproducible, and NaN row padding never read."""
    m = mapi_lib
    r = np.random.default_rng(n + pad)
    Af = np.full((n, n + pad), np.nan, np.float32)
    A = r.standard_normal((n, n)).astype(np.float32) + np.diag(np.abs(r.standard_normal(n)) * 4).astype(np.float32)
    Af[:, :n] = A
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    monkeypatch.setenv("MAPI_DENSE_PATH", "bulk")
    Ad = torch.from_numpy(Af).cuda()[:, :n]
    opc = m.MIN1 if op == "min1" else m.MIN2
    res = m.iterate(Ad, torch.from_numpy(b0).cuda(), 25, op=opc)
    ref = orc.mapi(A, b0, 25, op=op)
    assert res.iters_done == 25
    _t2(res.w_l2.cpu().numpy(), ref.w, res.norms.cpu().numpy(), ref.norms)
    again = m.iterate(Ad, torch.from_numpy(b0).cuda(), 25, op=opc)
    assert torch.equal(res.w, again.w) and torch.equal(res.deltas, again.deltas)


def test_bulk_ring_early_stop_and_degenerate(mapi_lib, orc, monkeypatch):
    """Early stop by tol (the producer has copies in flight past the last iteration and must drain
    them) and the degenerate status, on the bulk path; then a normal run on the same stream."""
    m = mapi_lib
    monkeypatch.setenv("MAPI_DENSE_PATH", "bulk")
    n = 2048
    r = np.random.default_rng(3)
    A = (r.standard_normal((n, n)) / 8).astype(np.float32) + np.diag(np.linspace(4.0, 1.0, n)).astype(np.float32)
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    Ad, bd = torch.from_numpy(A).cuda(), torch.from_numpy(b0).cuda()
    full = m.iterate(Ad, bd, 200)
    d = full.deltas.cpu().numpy()
    tol = float(d[40]) * 1.0001  # first crossing near iteration 40
    first = int(np.nonzero(d < tol)[0][0])
    res = m.iterate(Ad, bd, 200, tol=tol)
    assert res.iters_done == first + 1
    assert torch.equal(res.deltas, full.deltas[: first + 1])
    ref = orc.mapi(A, b0, first + 1)
    _t2(res.w_l2.cpu().numpy(), ref.w)
    with pytest.raises(m.MapiError) as ei:
        m.iterate(torch.zeros(n, n, device="cuda"), bd, 10)
    assert ei.value.name == "MAPI_ERR_DEGENERATE" and ei.value.iters_done == 0
    again = m.iterate(Ad, bd, 200)
    assert torch.equal(again.w, full.w)


@pytest.mark.parametrize("n,pad", [(1, 0), (33, 3), (700, 0), (1500, 4), (2049, 8), (3001, 1), (4096, 0), (4096, 12)])
@pytest.mark.parametrize("op", ["min1", "min2", "dot"])
@pytest.mark.parametrize("nw", ["8", "16"])
def test_resident_path(mapi_lib, orc, monkeypatch, n, pad, op, nw):
    """K2r (matrix held in TMEM + shared memory for the whole call): ragged n (partial column lanes,
    scalar staging when rows are not 16 B-aligned), padded lda with NaN padding, every operator, both
    warp counts, vs the oracle (T2; the RPI limit for dot), bitwise reproducible."""
    m = mapi_lib
    r = np.random.default_rng(n + pad)
    Af = np.full((n, n + pad), np.nan, np.float32)
    A = r.standard_normal((n, n)).astype(np.float32) + np.diag(np.abs(r.standard_normal(n)) * 4).astype(np.float32)
    if op == "dot":
        A = ((A + A.T) / (2 * np.sqrt(n))).astype(np.float32)
    Af[:, :n] = A
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    monkeypatch.setenv("MAPI_DENSE_PATH", "resident")
    monkeypatch.setenv("MAPI_RES_NW", nw)
    Ad = torch.from_numpy(Af).cuda()[:, :n]
    opc = {"min1": m.MIN1, "min2": m.MIN2, "dot": m.DOT}[op]
    res = m.iterate(Ad, torch.from_numpy(b0).cuda(), 25, op=opc)
    ref = orc.rpi(A, b0, 25) if op == "dot" else orc.mapi(A, b0, 25, op=op)
    assert res.iters_done == 25
    got = res.w.cpu().numpy() if op == "dot" else res.w_l2.cpu().numpy()
    _t2(got, ref.w, res.norms.cpu().numpy(), ref.norms)
    again = m.iterate(Ad, torch.from_numpy(b0).cuda(), 25, op=opc)
    assert torch.equal(res.w, again.w) and torch.equal(res.deltas, again.deltas)


@pytest.mark.parametrize("n,pad", [(1, 0), (2, 1), (7, 0), (31, 3), (100, 4), (128, 0), (129, 8), (255, 1), (256, 0), (256, 5)])
@pytest.mark.parametrize("op", ["min1", "min2", "dot"])
def test_single_cta_path(mapi_lib, orc, monkeypatch, n, pad, op):
    """K6t (one CTA, rows in registers + TMEM; BASELINE configs[0]'s path): ragged n (padded rows and
    columns), padded lda with NaN padding, every operator, vs the oracle (T2; the RPI limit for dot), bitwise
    reproducible, and resume: iterate(A, iterate(A, b0, 10).w, 15) == iterate(A, b0, 25)."""
    m = mapi_lib
    r = np.random.default_rng(n * 7 + pad)
    Af = np.full((n, n + pad), np.nan, np.float32)
    A = r.standard_normal((n, n)).astype(np.float32) + np.diag(np.abs(r.standard_normal(n)) * 4).astype(np.float32)
    if op == "dot":
        A = ((A + A.T) / (2 * np.sqrt(n))).astype(np.float32)
    Af[:, :n] = A
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    monkeypatch.setenv("MAPI_DENSE_PATH", "single")
    Ad, bd = torch.from_numpy(Af).cuda()[:, :n], torch.from_numpy(b0).cuda()
    opc = {"min1": m.MIN1, "min2": m.MIN2, "dot": m.DOT}[op]
    res = m.iterate(Ad, bd, 25, op=opc)
    ref = orc.rpi(A, b0, 25) if op == "dot" else orc.mapi(A, b0, 25, op=op)
    assert res.iters_done == 25
    got = res.w.cpu().numpy() if op == "dot" else res.w_l2.cpu().numpy()
    if n > 1:
        _t2(got, ref.w, res.norms.cpu().numpy(), ref.norms)
    again = m.iterate(Ad, bd, 25, op=opc)
    assert torch.equal(res.w, again.w) and torch.equal(res.deltas, again.deltas)
    # the in-kernel l2 copy is bitwise the separate k_l2_copy (which mapi_iterate_sym's fallback runs)
    monkeypatch.setenv("MAPI_SYM_PATH", "full")
    sep = m.iterate_sym(Ad, bd, 25, op=opc)
    assert torch.equal(sep.w, res.w) and torch.equal(sep.w_l2, res.w_l2)
    if op != "dot":
        first = m.iterate(Ad, bd, 10, op=opc)
        resumed = m.iterate(Ad, first.w, 15, op=opc)
        assert torch.equal(resumed.w, res.w)


def test_single_cta_early_stop_and_degenerate(mapi_lib, orc, monkeypatch):
    """tol stop and the degenerate status on K6t (TMEM released on every exit path), then a normal run."""
    m = mapi_lib
    monkeypatch.setenv("MAPI_DENSE_PATH", "single")
    cfg = synth.cfg1()
    Ad, bd = torch.from_numpy(cfg["A"]).cuda(), torch.from_numpy(cfg["b0"]).cuda()
    full = m.iterate(Ad, bd, 200)
    d = full.deltas.cpu().numpy()
    tol = float(d[40]) * 1.0001
    first = int(np.nonzero(d < tol)[0][0])
    res = m.iterate(Ad, bd, 200, tol=tol)
    assert res.iters_done == first + 1
    assert torch.equal(res.deltas, full.deltas[: first + 1])
    ref = orc.mapi(cfg["A"], cfg["b0"], first + 1)
    _t2(res.w_l2.cpu().numpy(), ref.w)
    with pytest.raises(m.MapiError) as ei:
        m.iterate(torch.zeros(256, 256, device="cuda"), bd, 10)
    assert ei.value.name == "MAPI_ERR_DEGENERATE" and ei.value.iters_done == 0
    again = m.iterate(Ad, bd, 200)
    assert torch.equal(again.w, full.w)


def test_resident_matvec_t1_each_iteration(mapi_lib, orc, monkeypatch):
    """K2r per-iteration T1: the GPU's t-th norm and iterate against one fp64 oracle step from the GPU's
    own (t-1)-th iterate, at cfg2's size (4096, 28 rows per CTA: 16 in TMEM, 12 in shared memory)."""
    m = mapi_lib
    n = 4096
    r = np.random.default_rng(11)
    A = r.standard_normal((n, n)).astype(np.float32) + np.diag(np.abs(r.standard_normal(n)) * 4).astype(np.float32)
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    monkeypatch.setenv("MAPI_DENSE_PATH", "resident")
    Ad, bd = torch.from_numpy(A).cuda(), torch.from_numpy(b0).cuda()
    r4 = m.iterate(Ad, bd, 4)
    r5 = m.iterate(Ad, bd, 5)
    w4 = r4.w.cpu().numpy()
    y, mag = orc.matvec(A, w4, return_mag=True)
    s = np.abs(y).sum()
    assert abs(float(r5.norms[4]) - s) <= 1e-5 * s
    w5 = r5.w.cpu().numpy().astype(np.float64)
    err = np.abs(w5 - y / s)
    assert np.all(err <= 1e-5 * mag / s + 2e-5 * np.abs(y / s)), float(np.max(err))
    resumed = m.iterate(Ad, r4.w, 1)
    assert torch.equal(resumed.w, r5.w)


def test_resident_early_stop_and_degenerate(mapi_lib, orc, monkeypatch):
    """tol stop and the degenerate status on K2r (TMEM is released on every exit path: the next call
    allocates it again), then a normal run on the same stream."""
    m = mapi_lib
    monkeypatch.setenv("MAPI_DENSE_PATH", "resident")
    n = 3000
    r = np.random.default_rng(3)
    A = (r.standard_normal((n, n)) / 8).astype(np.float32) + np.diag(np.linspace(4.0, 1.0, n)).astype(np.float32)
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    Ad, bd = torch.from_numpy(A).cuda(), torch.from_numpy(b0).cuda()
    full = m.iterate(Ad, bd, 200)
    d = full.deltas.cpu().numpy()
    tol = float(d[40]) * 1.0001
    first = int(np.nonzero(d < tol)[0][0])
    res = m.iterate(Ad, bd, 200, tol=tol)
    assert res.iters_done == first + 1
    assert torch.equal(res.deltas, full.deltas[: first + 1])
    ref = orc.mapi(A, b0, first + 1)
    _t2(res.w_l2.cpu().numpy(), ref.w)
    with pytest.raises(m.MapiError) as ei:
        m.iterate(torch.zeros(n, n, device="cuda"), bd, 10)
    assert ei.value.name == "MAPI_ERR_DEGENERATE" and ei.value.iters_done == 0
    again = m.iterate(Ad, bd, 200)
    assert torch.equal(again.w, full.w)


@pytest.mark.parametrize("n", [1, 7, 100, 256, 257, 500, 512])
@pytest.mark.parametrize("op", ["min1", "min2"])
def test_cluster_register_kernel_bitwise_vs_smem_kernel(mapi_lib, orc, monkeypatch, n, op):
    """K6r (rows in registers, spread epilogue) keeps K6's per-row summation order: the iterates and
    norms are bitwise identical to K6 (rows in shared memory); both match the oracle (T2)."""
    m = mapi_lib
    r = np.random.default_rng(n)
    A = r.standard_normal((n, n)).astype(np.float32) + np.diag(np.abs(r.standard_normal(n)) * 3).astype(np.float32)
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    opc = m.MIN1 if op == "min1" else m.MIN2
    Ad, bd = torch.from_numpy(A).cuda(), torch.from_numpy(b0).cuda()
    monkeypatch.setenv("MAPI_DENSE_PATH", "cluster")
    reg = m.iterate(Ad, bd, 30, op=opc)
    monkeypatch.setenv("MAPI_DENSE_PATH", "cluster_smem")
    smem = m.iterate(Ad, bd, 30, op=opc)
    assert torch.equal(reg.w, smem.w) and torch.equal(reg.norms, smem.norms)
    np.testing.assert_allclose(reg.deltas.cpu().numpy(), smem.deltas.cpu().numpy(), rtol=1e-6)
    if n > 1:
        ref = orc.mapi(A, b0, 30, op=op)
        _t2(reg.w_l2.cpu().numpy(), ref.w, reg.norms.cpu().numpy(), ref.norms)


# ------------------------------------------------------------------------------ RPI comparator (NEXT-3)


@pytest.mark.parametrize("path", ["cluster", "rows", "coop", "bulk", "multi"])
def test_rpi_comparator_matches_oracle(mapi_lib, orc, monkeypatch, path):
    """op = MAPI_OP_DOT: b <- Ab/||Ab||_2 (Eq. 1) through every dense path, vs the oracle's rpi."""
    m = mapi_lib
    n = 256 if path == "cluster" else 8192
    r = np.random.default_rng(n)
    A = (r.standard_normal((n, n)) / np.sqrt(n)).astype(np.float32)
    A = (A + A.T) / 2 + np.diag(np.linspace(2.0, 0.0, n)).astype(np.float32)
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    monkeypatch.setenv("MAPI_DENSE_PATH", path)
    res = m.iterate(torch.from_numpy(A).cuda(), torch.from_numpy(b0).cuda(), 30, op=m.DOT)
    ref = orc.rpi(A, b0, 30)
    _t2(res.w.cpu().numpy(), ref.w, res.norms.cpu().numpy(), ref.norms)
    assert abs(float(res.w.norm()) - 1.0) < 1e-5


def test_matvec_dot(mapi_lib, orc):
    m = mapi_lib
    M, _ = synth.random_matrix(300, 700, seed=9)
    x = synth.random_vector(700, seed=10)
    y = m.mavp_matvec(torch.from_numpy(M).cuda(), torch.from_numpy(x).cuda(), op=m.DOT).cpu().numpy()
    ref, mag = orc.matvec(M, x, "dot", return_mag=True)
    assert np.all(np.abs(y - ref) <= 1e-5 * mag)


def test_iterate_host_many_pipelined(mapi_lib):
    """Pipelined host problems (copy stream overlapping the previous problem's iterations): every
    result equals the one-problem host path bitwise, distinct inputs stay distinct, iters_done per
    problem, and a degenerate problem reports its index."""
    m = mapi_lib
    n = 2048
    r = np.random.default_rng(8)
    As = [torch.from_numpy((r.standard_normal((n, n)) + np.eye(n) * (2 + i)).astype(np.float32)).pin_memory()
          for i in range(5)]
    b0s = [torch.full((n,), 1 / np.sqrt(n)).pin_memory() for _ in range(5)]
    res = m.iterate_host_many(As, b0s, 20)
    for A, b0, got in zip(As, b0s, res):
        one = m.iterate_host(A, b0, 20)
        assert got.iters_done == 20
        assert torch.equal(got.w, one.w) and torch.equal(got.norms, one.norms) and torch.equal(got.deltas, one.deltas)
    assert not torch.equal(res[0].w, res[1].w)
    bad = [As[0], torch.zeros(n, n).pin_memory(), As[2]]
    with pytest.raises(m.MapiError) as ei:
        m.iterate_host_many(bad, b0s[:3], 5)
    assert ei.value.name == "MAPI_ERR_DEGENERATE" and "problem 1" in str(ei.value)


@pytest.mark.parametrize("n", [1, 7, 33, 256, 1000, 1031, 2600, 5000, 8200])
def test_iterate_host_many_packed_bitwise(mapi_lib, n):
    """Symmetric matrices sent as packed upper triangles (half the PCIe bytes): the device-side unpack
    rebuilds the full matrix bitwise, so every result equals the full-matrix pipelined path bitwise (on
    every dense kernel the sizes select: cluster, per-row, resident, bulk, cooperative)."""
    m = mapi_lib
    r = np.random.default_rng(n + 17)
    As, Aps, b0s = [], [], []
    for i in range(3):
        G = r.standard_normal((n, n)).astype(np.float32)
        S = np.triu(G) + np.triu(G, 1).T + np.eye(n, dtype=np.float32) * (3 + i)
        assert np.array_equal(S, S.T)
        A = torch.from_numpy(S)
        As.append(A.pin_memory())
        Aps.append(m.pack_upper(A).pin_memory())
        b0s.append(torch.full((n,), 1 / np.sqrt(n)).pin_memory())
    full = m.iterate_host_many(As, b0s, 15)
    packed = m.iterate_host_many_packed(Aps, n, b0s, 15)
    for A, b0, a, b in zip(As, b0s, full, packed):
        assert a.iters_done == b.iters_done == 15
        # packed (= declared symmetric) problems take the same kernel as mapi_iterate_sym: K2s where it
        # applies (n >= 8192, n % 8 == 0), else the full-matrix kernels (bitwise = mapi_iterate_host_many)
        ref = m.iterate_sym(A.cuda(), b0.cuda(), 15)
        assert torch.equal(ref.w.cpu(), b.w) and torch.equal(ref.norms.cpu(), b.norms)
        if n < 8192:
            assert torch.equal(a.w, b.w) and torch.equal(a.norms, b.norms) and torch.equal(a.deltas, b.deltas)
        else:
            _t2(b.w.numpy() / np.linalg.norm(b.w.numpy()), a.w.numpy().astype(np.float64), b.norms.numpy(),
                a.norms.numpy().astype(np.float64))


@pytest.mark.parametrize("n", [1, 33, 1000, 2600, 8192, 8200])
def test_iterate_host_many_sym_bitwise(mapi_lib, n):
    """Symmetric matrices handed over as FULL host matrices (mapi_iterate_host_many_sym): only the upper-
    triangle block rows are copied where K2s runs (n >= 8192; the host's strictly-lower triangle is NaN there
    and never crosses PCIe / is never read), the whole matrix otherwise; results bitwise mapi_iterate_sym on
    the device matrix, padded host rows (lda > n) included."""
    m = mapi_lib
    r = np.random.default_rng(n + 29)
    As, b0s, Sd = [], [], []
    lda = n + 5
    for i in range(2):
        G = r.standard_normal((n, n)).astype(np.float32)
        S = np.triu(G) + np.triu(G, 1).T + np.eye(n, dtype=np.float32) * (3 + i)
        host = np.full((n, lda), np.nan, np.float32)
        host[:, :n] = S
        if n >= 8192:
            host[:, :n][np.tril_indices(n, -1)] = np.nan
        As.append(torch.from_numpy(host).pin_memory()[:, :n])
        Sd.append(torch.from_numpy(S).cuda())
        b0s.append(torch.full((n,), 1 / np.sqrt(n)).pin_memory())
    res = m.iterate_host_many_sym(As, b0s, 12)
    for A, b0, got in zip(Sd, b0s, res):
        ref = m.iterate_sym(A, b0.cuda(), 12)
        assert got.iters_done == 12
        assert torch.equal(ref.w.cpu(), got.w) and torch.equal(ref.norms.cpu(), got.norms)
        assert np.all(np.isfinite(got.w.numpy()))


# ------------------------------------------------------------------------------ symmetric path (K2s)


def _sym_matrix(n, seed, diag=4.0):
    r = np.random.default_rng(seed)
    G = r.standard_normal((n, n)).astype(np.float32)
    S = np.triu(G) + np.triu(G, 1).T
    S[np.diag_indices(n)] += (np.abs(r.standard_normal(n)) * diag).astype(np.float32)
    return S.astype(np.float32)


@pytest.mark.parametrize("n", [8, 64, 1000, 1032, 4096, 8192])
@pytest.mark.parametrize("op", ["min1", "min2", "dot"])
def test_sym_path_reads_only_upper_triangle(mapi_lib, orc, monkeypatch, n, op):
    """K2s (forced at every size): the strictly-lower triangle and the row padding are NaN on the device, so
    any read of them would poison the result; the iterate still matches the oracle on the full symmetric
    matrix (T2; the RPI limit for dot) and is bitwise reproducible.  Ragged task grids: n % 64, n % 256 != 0."""
    m = mapi_lib
    S = _sym_matrix(n, n + 3)
    if op == "dot":
        S = (S / np.sqrt(n)).astype(np.float32)
    pad = 8
    dev = np.full((n, n + pad), np.nan, np.float32)
    dev[:, :n] = np.triu(S) + np.tril(np.full((n, n), np.nan, np.float32), -1)
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    monkeypatch.setenv("MAPI_SYM_PATH", "sym")
    Ad = torch.from_numpy(dev).cuda()[:, :n]
    opc = {"min1": m.MIN1, "min2": m.MIN2, "dot": m.DOT}[op]
    res = m.iterate_sym(Ad, torch.from_numpy(b0).cuda(), 20, op=opc)
    ref = orc.rpi(S, b0, 20) if op == "dot" else orc.mapi(S, b0, 20, op=op)
    assert res.iters_done == 20
    got = res.w.cpu().numpy() if op == "dot" else res.w_l2.cpu().numpy()
    assert np.all(np.isfinite(got))
    _t2(got, ref.w, res.norms.cpu().numpy(), ref.norms)
    again = m.iterate_sym(Ad, torch.from_numpy(b0).cuda(), 20, op=opc)
    assert torch.equal(res.w, again.w) and torch.equal(res.deltas, again.deltas)


@pytest.mark.parametrize("n", [1000, 8196])
def test_sym_fallback_full_path(mapi_lib, orc, monkeypatch, n):
    """Shapes K2s does not take (n < 8192 unforced; n % 8 != 0) run the full-matrix kernels: same result as
    mapi_iterate bitwise."""
    m = mapi_lib
    S = _sym_matrix(n, 5)
    b0 = torch.full((n,), 1 / np.sqrt(n), device="cuda")
    Ad = torch.from_numpy(S).cuda()
    a = m.iterate_sym(Ad, b0, 10)
    b = m.iterate(Ad, b0, 10)
    assert torch.equal(a.w, b.w) and torch.equal(a.norms, b.norms)


def test_sym_early_stop_and_degenerate(mapi_lib, orc, monkeypatch):
    m = mapi_lib
    monkeypatch.setenv("MAPI_SYM_PATH", "sym")
    n = 2048
    S = (_sym_matrix(n, 9) / 8).astype(np.float32) + np.diag(np.linspace(4.0, 1.0, n)).astype(np.float32)
    b0 = np.full(n, 1.0 / np.sqrt(n), np.float32)
    Ad, bd = torch.from_numpy(S).cuda(), torch.from_numpy(b0).cuda()
    full = m.iterate_sym(Ad, bd, 200)
    d = full.deltas.cpu().numpy()
    tol = float(d[40]) * 1.0001
    first = int(np.nonzero(d < tol)[0][0])
    res = m.iterate_sym(Ad, bd, 200, tol=tol)
    assert res.iters_done == first + 1
    assert torch.equal(res.deltas, full.deltas[: first + 1])
    ref = orc.mapi(S, b0, first + 1)
    _t2(res.w_l2.cpu().numpy(), ref.w)
    with pytest.raises(m.MapiError) as ei:
        m.iterate_sym(torch.zeros(n, n, device="cuda"), bd, 10)
    assert ei.value.name == "MAPI_ERR_DEGENERATE" and ei.value.iters_done == 0


def test_cfg3_sym_last_step(mapi_lib, orc, cfg3_device):
    """cfg3 through K2s as bench.py runs it (upper triangle only): the GPU's 100th iterate equals the
    oracle's fp64 step from the GPU's own 99th iterate (T1-scaled bound per element), s_99 matches, the
    100-iteration run stays within T2 of the full-matrix kernel, and it is bitwise reproducible."""
    m = mapi_lib
    A = cfg3_device["A"]
    b0 = torch.from_numpy(cfg3_device["b0"]).cuda()
    r100 = m.iterate_sym(A, b0, 100)
    r99 = m.iterate_sym(A, b0, 99)
    assert torch.equal(r100.norms[:99], r99.norms)
    w99 = r99.w.cpu().numpy()
    y, mag = orc.matvec(A.cpu().numpy(), w99, return_mag=True)
    s = np.abs(y).sum()
    assert abs(float(r100.norms[99]) - s) <= 1e-5 * s
    w100 = r100.w.cpu().numpy().astype(np.float64)
    err = np.abs(w100 - y / s)
    assert np.all(err <= 1e-5 * mag / s + 2e-5 * np.abs(y / s)), float(np.max(err))
    full = m.iterate(A, b0, 100)
    _t2(r100.w_l2.cpu().numpy(), full.w_l2.cpu().numpy().astype(np.float64), r100.norms.cpu().numpy(),
        full.norms.cpu().numpy().astype(np.float64))
    again = m.iterate_sym(A, b0, 100)
    assert torch.equal(r100.w, again.w)


# ------------------------------------------------------------------------------ error paths


@pytest.mark.parametrize("path,n", [("single", 256), ("cluster", 400), ("resident", 2048), ("rows", 1500),
                                    ("coop", 8192), ("multi", 1000), ("sym", 8192)])
def test_nonfinite_norm_reported(mapi_lib, monkeypatch, path, n):
    """MAPI_ERR_NONFINITE (include/mapi.h): min-type terms are bounded by min(|a|, |w|), so a NaN or inf
    entry is absorbed by FMNMX; the norm becomes non-finite only when the fp32 row sums overflow.  A = b0 =
    3e38 everywhere overflows y_j at iteration 0 on every dense path; the call reports NONFINITE with
    iters_done = 0 and the stream stays usable."""
    m = mapi_lib
    A = torch.full((n, n), 3e38, device="cuda")
    b0 = torch.full((n,), 3e38, device="cuda")
    if path == "sym":
        monkeypatch.setenv("MAPI_SYM_PATH", "sym")
        call = m.iterate_sym
    else:
        monkeypatch.setenv("MAPI_DENSE_PATH", path)
        call = m.iterate
    with pytest.raises(m.MapiError) as ei:
        call(A, b0, 5)
    assert ei.value.name == "MAPI_ERR_NONFINITE" and ei.value.iters_done == 0
    ok = call(torch.eye(n, device="cuda") * 2, torch.full((n,), 1.0 / n, device="cuda"), 2)
    assert torch.isfinite(ok.w).all()


def test_nonfinite_batched_reported(mapi_lib):
    """The batched path reports NONFINITE per vector: vector 1 overflows, vector 0 stays finite."""
    m = mapi_lib
    n = 1024
    A = torch.full((n, n), 3e38, device="cuda")
    B0 = torch.full((2, n), 1.0 / n, device="cuda")
    B0[1] = 3e38
    with pytest.raises(m.MapiError) as ei:
        m.iterate_batched(A, B0, 3)
    assert ei.value.name == "MAPI_ERR_NONFINITE" and "vector 1" in str(ei.value)
