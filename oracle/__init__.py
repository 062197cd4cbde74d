"""fp64 CPU oracle for the MAPI / MAVP hot path (arXiv 2110.12065) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  It shares no code with the CUDA library
(``paper_2110_12065_b200``) and never imports it; the CUDA library never imports this.

``oracle.c`` holds the arithmetic (plain loops, fp64, rows summed in index order,
``-O2 -fno-fast-math -ffp-contract=off``); this module is ctypes marshalling only.
``brute.py`` is the literal-definition brute force used to pin ``oracle.c``.

Citation keys: ``P:n`` = PAPER.md line n; ``S:n`` = SPEC.md line n.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

MIN1, MIN2, DIAMOND, DOT = 0, 1, 2, 3
NORM_L1, NORM_L2 = 1, 2
OK, ERR_BAD_PARAM, ERR_DEGENERATE, ERR_NEGATIVE, ERR_NONFINITE = 0, 3, 4, 5, 6

_OPS = {"min1": MIN1, "min2": MIN2, "diamond": DIAMOND, "dot": DOT}


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (OpenMP over rows only)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC",
           "-shared", "-std=c11", "-o", tmp, _SRC, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, dbl, cint = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_int
        lib.orc_mavp_dot.argtypes = [cint, P, P, i64]
        lib.orc_mavp_dot.restype = dbl
        lib.orc_matvec_f32.argtypes = [cint, P, i64, i64, i64, P, P, P]
        lib.orc_matvec_f32.restype = None
        lib.orc_matvec_f64.argtypes = [cint, P, i64, i64, i64, P, P, P]
        lib.orc_matvec_f64.restype = None
        lib.orc_power_iterate.argtypes = [cint, cint, P, cint, i64, i64, P, i32, dbl, P, P, P, P,
                                          ctypes.POINTER(i32)]
        lib.orc_power_iterate.restype = cint
        lib.orc_matmat_f32.argtypes = [cint, P, i64, i64, i64, P, i64, i64, dbl, P]
        lib.orc_matmat_f32.restype = None
        lib.orc_outer_apply.argtypes = [cint, P, i64, i64, i64, P, i64, i64, cint, P, i64]
        lib.orc_outer_apply.restype = None
        lib.orc_outer_apply_rows.argtypes = [cint, P, i64, i64, i64, P, i64, i64, cint, P, i64, P, i64]
        lib.orc_outer_apply_rows.restype = None
        lib.orc_deflate.argtypes = [P, i64, i64, P, i32, P]
        lib.orc_deflate.restype = None
        lib.orc_pca_topk.argtypes = [cint, P, i64, i64, i32, i32, P, P, P, P, P]
        lib.orc_pca_topk.restype = cint
        lib.orc_rank_csr.argtypes = [i64, i64, P, P, dbl, P, i32, dbl, P, P, P,
                                     ctypes.POINTER(i32)]
        lib.orc_rank_csr.restype = cint
        lib.orc_rank_csr_op.argtypes = [cint, i64, i64, P, P, dbl, P, i32, dbl, P, P, P, ctypes.POINTER(i32)]
        lib.orc_rank_csr_op.restype = cint
        lib.orc_minibatch_mapi.argtypes = [P, i64, i64, i64, P, i32, i32, dbl, P, cint, P, P, P, ctypes.POINTER(i32),
                                           P, P]
        lib.orc_minibatch_mapi.restype = cint
        lib.orc_num_threads.argtypes = []
        lib.orc_num_threads.restype = cint
        lib.orc_set_num_threads.argtypes = [cint]
        lib.orc_set_num_threads.restype = None
        _lib = lib
        return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _op(op) -> int:
    return _OPS[op] if isinstance(op, str) else int(op)


def num_threads() -> int:
    return int(_load().orc_num_threads())


def set_num_threads(n: int) -> None:
    _load().orc_set_num_threads(int(n))


def mavp_dot(w, x, op="min1") -> float:
    """w^T (op) x — Eq.(3) min1, Eq.(4) min2, Eq.(9) diamond, dot."""
    w, x = _f64(w), _f64(x)
    if w.shape != x.shape or w.ndim != 1:
        raise ValueError(f"dimension mismatch: {w.shape} vs {x.shape}")
    return float(_load().orc_mavp_dot(_op(op), _ptr(w), _ptr(x), w.size))


def _as_f32_matrix(A):
    A = np.asarray(A)
    if A.dtype != np.float32:
        raise TypeError("oracle matrices are the fp32 input bytes (dtype float32)")
    if A.ndim == 2 and A.size == 0:
        return np.ascontiguousarray(A), max(1, A.shape[1])
    if A.ndim == 2 and A.flags.c_contiguous:
        return A, A.shape[1]
    if A.ndim != 2 or A.strides[1] != 4:
        raise ValueError("A must be a 2-D row-major float32 array")
    lda = A.strides[0] // 4
    return A, lda


def matvec(A, x, op="min1", return_mag=False):
    """y_j = row_j(A)^T (op) x  (matrix extension, reading Q6/Q7).

    A is fp32 (the same bytes the GPU sees) or fp64; x is promoted to fp64.
    Returns y (fp64) and, if requested, mag_j = sum_k |term_jk| (tolerance scale T1).
    """
    A = np.asarray(A)
    x = _f64(x)
    n_rows, n_cols = A.shape
    if x.shape != (n_cols,):
        raise ValueError(f"dimension mismatch: A has {n_cols} columns, x has {x.shape}")
    y = np.empty(n_rows, np.float64)
    mag = np.empty(n_rows, np.float64)
    lib = _load()
    if A.dtype == np.float64:
        if A.strides[1] != 8:
            A = np.ascontiguousarray(A)
        lib.orc_matvec_f64(_op(op), _ptr(A), n_rows, n_cols, A.strides[0] // 8, _ptr(x),
                           _ptr(y), _ptr(mag))
    else:
        A, lda = _as_f32_matrix(A)
        lib.orc_matvec_f32(_op(op), _ptr(A), n_rows, n_cols, lda, _ptr(x), _ptr(y), _ptr(mag))
    return (y, mag) if return_mag else y


class IterResult:
    """Result of a power iteration: w (l1- or l2-unit iterate), w_l2, norms, deltas, status."""

    def __init__(self, status, w, w_l2, norms, deltas, iters_done):
        self.status, self.w, self.w_l2 = status, w, w_l2
        self.norms, self.deltas, self.iters_done = norms, deltas, iters_done

    def __repr__(self):
        return f"IterResult(status={self.status}, iters_done={self.iters_done})"


def power_iterate(A, b0, iters, tol=0.0, op="min1", norm=None) -> IterResult:
    """Algorithm 1 (MAPI) for min-type ops, Eq.(1) RPI for op='dot'.

    norm defaults to l1 for MAVP ops (Eq. 8) and l2 for 'dot' (Eq. 1).
    """
    opc = _op(op)
    if norm is None:
        norm = NORM_L2 if opc == DOT else NORM_L1
    A = np.asarray(A)
    n = A.shape[0]
    if A.ndim != 2 or A.shape[1] != n:
        raise ValueError(f"A must be square, got {A.shape}")
    if A.dtype == np.float64:
        A = np.ascontiguousarray(A)
        lda, is64 = n, 1
    else:
        A, lda = _as_f32_matrix(A)
        is64 = 0
    b0 = _f64(b0)
    if b0.shape != (n,):
        raise ValueError(f"dimension mismatch: A is {n}x{n}, b0 has {b0.shape}")
    w = np.zeros(n)
    wl2 = np.zeros(n)
    norms = np.zeros(iters)
    deltas = np.zeros(iters)
    done = ctypes.c_int32(0)
    st = _load().orc_power_iterate(opc, norm, _ptr(A), is64, n, lda, _ptr(b0), int(iters),
                                   float(tol), _ptr(w), _ptr(wl2), _ptr(norms), _ptr(deltas),
                                   ctypes.byref(done))
    k = done.value
    return IterResult(st, w, wl2, norms[:k], deltas[:k], k)


def mapi(A, b0, iters, tol=0.0, op="min1") -> IterResult:
    """MAPI, Eq.(8) / Algorithm 1: w <- (A (op) w) / ||A (op) w||_1."""
    if _op(op) == DOT:
        raise ValueError("mapi() takes a multiplication-avoiding operator; use rpi() for 'dot'")
    return power_iterate(A, b0, iters, tol, op, NORM_L1)


def rpi(A, b0, iters, tol=0.0) -> IterResult:
    """Regular power iteration, Eq.(1): b <- Ab / ||Ab||_2."""
    return power_iterate(A, b0, iters, tol, "dot", NORM_L2)


def matmat(A, B, op="min1", d=1.0) -> np.ndarray:
    """C[i][j] = (row_i(A) (op) row_j(B)) / d — matrix extension; A, B fp32 row-major."""
    A, lda = _as_f32_matrix(A)
    B, ldb = _as_f32_matrix(B)
    m, K = A.shape
    p, K2 = B.shape
    if K != K2:
        raise ValueError(f"dimension mismatch: A is {m}x{K}, B is {p}x{K2}")
    C = np.empty((m, p), np.float64)
    _load().orc_matmat_f32(_op(op), _ptr(A), m, K, lda, _ptr(B), p, ldb, float(d), _ptr(C))
    return C


def min_covariance(V, divisor=None, op="min1") -> np.ndarray:
    """Min-covariance (1/d) V (+) V^T of mean-removed samples V (pixels x N): d = N - 1 as in Alg. 2
    step 4 by default; d = N reproduces Eq. (5)."""
    V = np.asarray(V)
    d = (V.shape[1] - 1) if divisor is None else divisor
    return matmat(V, V, op, d)


def outer_apply(W, X, op="min1", subtract=False) -> np.ndarray:
    """Y = (W (op) W^T) X, or X - (W (op) W^T) X: Alg. 2 steps 8 / 6, regular product."""
    W = np.asarray(W, np.float32)
    if W.ndim == 1:
        W = W[:, None]
    W, ldw = _as_f32_matrix(np.ascontiguousarray(W))
    X = np.asarray(X, np.float32)
    vec = X.ndim == 1
    if vec:
        X = X[:, None]
    X, ldx = _as_f32_matrix(np.ascontiguousarray(X))
    M, r = W.shape
    if X.shape[0] != M:
        raise ValueError(f"dimension mismatch: W has {M} rows, X has {X.shape[0]}")
    q = X.shape[1]
    Y = np.empty((M, q), np.float64)
    _load().orc_outer_apply(_op(op), _ptr(W), M, r, ldw, _ptr(X), q, ldx, 1 if subtract else 0, _ptr(Y), q)
    return Y[:, 0] if vec else Y


def outer_apply_rows(W, X, rows, op="min1", subtract=False) -> np.ndarray:
    """Rows `rows` of outer_apply(W, X, op, subtract) (full-size checks on sampled rows)."""
    W = np.asarray(W, np.float32)
    if W.ndim == 1:
        W = W[:, None]
    W, ldw = _as_f32_matrix(np.ascontiguousarray(W))
    X, ldx = _as_f32_matrix(np.ascontiguousarray(np.asarray(X, np.float32)))
    rows = np.ascontiguousarray(np.asarray(rows, np.int64))
    M, r = W.shape
    q = X.shape[1]
    Y = np.empty((rows.size, q), np.float64)
    _load().orc_outer_apply_rows(_op(op), _ptr(W), M, r, ldw, _ptr(X), q, ldx, 1 if subtract else 0, _ptr(rows),
                                 rows.size, _ptr(Y), q)
    return Y


def mavp_deflate(C, w, op="min1") -> np.ndarray:
    """Alg. 2 step 6: C - (w (op) w^T) C, the scalar-MAVP outer product times C."""
    return outer_apply(w, C, op, subtract=True)


def reconstruct(W, V, op="min1"):
    """Alg. 2 steps 3 and 8: m = mean(V, 2); v_hat_i = (W (op) W^T)(v_i - m) + m for every
    column i of V (pixels x N).  Returns (V_hat fp64, m)."""
    V64 = np.asarray(V, np.float64)
    m = V64.mean(axis=1)
    Xc = (V64 - m[:, None]).astype(np.float32)
    return outer_apply(W, Xc, op) + m[:, None], m


def psnr(ref, test) -> float:
    """10 log10(1 / MSE), pixels in [0, 1] (peak 1)."""
    mse = float(np.mean((np.asarray(ref, np.float64) - np.asarray(test, np.float64)) ** 2))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(1.0 / mse)


def deflate(C, P, i) -> np.ndarray:
    """D_i = (I - sum_{m<i} p_m p_m^T) C, fp64 result, C fp32."""
    C, ldc = _as_f32_matrix(C)
    n = C.shape[0]
    P = _f64(P).reshape(-1, n)
    D = np.empty((n, n), np.float64)
    _load().orc_deflate(_ptr(C), n, ldc, _ptr(P), int(i), _ptr(D))
    return D


class PcaResult:
    def __init__(self, status, P, norms, deltas, iters_done):
        self.status, self.P, self.norms, self.deltas, self.iters_done = (
            status, P, norms, deltas, iters_done)


def pca_topk(C, k, iters, b0, op="min1") -> PcaResult:
    """Top-k principal vectors by MAPI with L2 deflation (BJ configs[1])."""
    C, ldc = _as_f32_matrix(C)
    n = C.shape[0]
    b0 = _f64(b0)
    P = np.zeros((k, n))
    norms = np.zeros((k, iters))
    deltas = np.zeros((k, iters))
    done = np.zeros(k, np.int32)
    st = _load().orc_pca_topk(_op(op), _ptr(C), n, ldc, int(k), int(iters), _ptr(b0), _ptr(P),
                              _ptr(norms), _ptr(deltas), _ptr(done))
    return PcaResult(st, P, norms, deltas, done)


def rank_csr(n, row_ptr, col_idx, alpha=0.85, b0=None, max_iters=200, tol=1e-7, op="min1") -> IterResult:
    """MAPI ranking on G = alpha M + (1-alpha)/n 1 (Eq. 13), CSR by destination.
    op="dot": the regular PageRank power iteration G w (RPI arm of Sec. 3.3, reading R13)."""
    row_ptr = np.ascontiguousarray(np.asarray(row_ptr, dtype=np.int64))
    col_idx = np.ascontiguousarray(np.asarray(col_idx, dtype=np.int32))
    if row_ptr.shape != (n + 1,):
        raise ValueError("row_ptr must have n+1 entries")
    nnz = int(row_ptr[-1])
    if b0 is None:
        b0 = np.full(n, 1.0 / n)
    b0 = _f64(b0)
    w = np.zeros(n)
    wl2 = np.zeros(n)
    deltas = np.zeros(max_iters)
    done = ctypes.c_int32(0)
    st = _load().orc_rank_csr_op(_op(op), n, nnz, _ptr(row_ptr), _ptr(col_idx), float(alpha), _ptr(b0),
                                 int(max_iters), float(tol), _ptr(w), _ptr(wl2), _ptr(deltas),
                                 ctypes.byref(done))
    k = done.value
    return IterResult(st, w, wl2, None, deltas[:k], k)


def minibatch_mapi(X, batch, beta, w0, gram="min1", w_prev0=None) -> IterResult:
    """Algorithm 3: mini-batch MAPI with momentum on the samples X (N x D, fp64).  batch: T x s
    row indices (the i.i.d. draws of step 3, an input); beta: momentum; w0: the start (step 1, used as
    given); gram: 'min1' (A~_i = x_i (.) x_i^T, the paper's A = X^T (.) X, reading R14) or 'dot'
    (x_i x_i^T).  Returns w (l1-unit w_T), w_l2 (Alg. 3 line 7), norms[t] = ||w_{t+1}||_1 before
    normalisation; deltas are not defined for Alg. 3 (empty).  w_prev0: the momentum vector to continue a run
    from (default: the paper's w_{-1} = 0); the result's w_prev is the momentum vector after the last step."""
    X = np.ascontiguousarray(np.asarray(X, np.float64))
    N, D = X.shape
    batch = np.ascontiguousarray(np.asarray(batch, np.int64))
    if batch.ndim != 2:
        raise ValueError("batch must be T x s")
    T, s = batch.shape
    w0 = _f64(w0)
    if w0.shape != (D,):
        raise ValueError(f"w0 must have D = {D} entries")
    w, wl2, norms, wprev = np.zeros(D), np.zeros(D), np.zeros(T), np.zeros(D)
    if w_prev0 is not None:
        w_prev0 = _f64(w_prev0)
        if w_prev0.shape != (D,):
            raise ValueError(f"w_prev0 must have D = {D} entries")
    done = ctypes.c_int32(0)
    st = _load().orc_minibatch_mapi(_ptr(X), N, D, D, _ptr(batch), int(s), int(T), float(beta), _ptr(w0),
                                    _op(gram), _ptr(w), _ptr(wl2), _ptr(norms), ctypes.byref(done),
                                    None if w_prev0 is None else _ptr(w_prev0), _ptr(wprev))
    if st == ERR_BAD_PARAM:
        raise ValueError("minibatch_mapi: bad parameters (empty input or a batch index out of range)")
    k = done.value
    res = IterResult(st, w, wl2, norms[:k], np.zeros(0), k)
    res.w_prev = wprev
    return res


def rank_order(scores) -> np.ndarray:
    """Indices sorted by descending score, ties by ascending index."""
    scores = np.asarray(scores)
    return np.lexsort((np.arange(scores.size), -scores))


def topk_overlap(a, b, k) -> int:
    """|first k of a  ∩  first k of b| ("7 common top-10 ranks")."""
    return len(set(list(a)[:k]) & set(list(b)[:k]))
