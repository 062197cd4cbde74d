"""paper_2110_12065_b200 — B200 (sm_100a) MAPI / MAVP hot path, Python binding of libmapi.so.

Thin ctypes marshalling over the C ABI declared in ``include/mapi.h`` (same names):
torch tensors supply device pointers and streams; workspaces are torch allocations.
Every step of the hot path runs in the library's CUDA kernels.  There is no CPU fallback:
if ``libmapi.so`` is missing or no sm_100 GPU is present, calls raise.

Citation keys: ``P:n`` = PAPER.md line n (arXiv 2110.12065 LaTeX source).
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass
from typing import Optional

from ._build import LIB as _LIB_PATH
from ._build import build  # noqa: F401  (re-exported: compile in-tree)

__all__ = ["load", "build", "MapiError", "mavp_matvec", "mavp_matmat", "min_covariance", "center_rows", "mavp_deflate",
           "mavp_reconstruct", "iterate", "iterate_host", "iterate_batched",
           "pca_topk", "csr_prepare", "rank_csr", "workspace_size", "launch_count", "set_profiling",
           "last_kernel_ms", "MIN1", "MIN2", "DOT", "iterate_host_many", "iterate_host_many_packed", "iterate_host_many_sym", "pack_upper", "iterate_sym", "csr_reorder", "csr_permute",
           "csr_plan", "rank_csr_plan", "CsrPlan", "PlanInfo", "minibatch"]

MIN1, MIN2, DOT = 0, 1, 2  # DOT: regular product of Eq. (1), the RPI comparator
(WS_MATVEC, WS_ITERATE, WS_ITERATE_BATCHED, WS_PCA_TOPK, WS_CSR_PREPARE, WS_RANK_CSR, WS_ITERATE_HOST,
 WS_MAVP_DEFLATE, WS_RECONSTRUCT, WS_ITERATE_SHARDED, WS_ITERATE_HOST_MANY,
 WS_ITERATE_HOST_MANY_PACKED, WS_ITERATE_SYM, WS_CSR_REORDER, WS_CSR_PLAN, WS_CSR_PLAN_BUILD,
 WS_RANK_CSR_PLAN, WS_ITERATE_HOST_MANY_SYM, WS_MINIBATCH, WS_RANK_CSR_SHARD) = range(20)
STATUS = {0: "MAPI_OK", 1: "MAPI_ERR_NULL", 2: "MAPI_ERR_SHAPE", 3: "MAPI_ERR_BAD_PARAM",
          4: "MAPI_ERR_DEGENERATE", 5: "MAPI_ERR_NEGATIVE", 6: "MAPI_ERR_NONFINITE",
          7: "MAPI_ERR_WORKSPACE", 8: "MAPI_ERR_CUDA"}

_lock = threading.Lock()
_lib = None


class MapiError(RuntimeError):
    def __init__(self, status: int, message: str, iters_done: Optional[int] = None):
        self.status = status
        self.name = STATUS.get(status, str(status))
        self.iters_done = iters_done
        super().__init__(f"{self.name}: {message}")


def load():
    """Load libmapi.so (built in-tree by build()); raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} not found: run paper_2110_12065_b200.build() "
                              "(nvcc, sm_100a) first — there is no CPU fallback")
        lib = ctypes.CDLL(_LIB_PATH)
        P, i64, i32, f32, sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float,
                                ctypes.c_size_t)
        st = ctypes.c_int
        sig = {
            "mapi_mavp_matvec": (st, [i32, P, i64, i64, i64, P, P, P]),
            "mapi_mavp_matmat": (st, [i32, P, i64, i64, i64, P, i64, i64, f32, P, i64, P]),
            "mapi_center_rows": (st, [P, i64, i64, i64, P, i64, P, P]),
            "mapi_normalize": (st, [i32, P, i64, P, P, P, P, P]),
            "mapi_matvec_normalized": (st, [i32, P, i64, i64, i64, P, P, P, P, P, P, P, P]),
            "mapi_mavp_deflate": (st, [i32, P, i64, i64, P, P, i64, P, sz, P]),
            "mapi_mavp_reconstruct": (st, [i32, P, i64, i32, i64, P, i64, i64, P, i64, P, P, sz, P]),
            "mapi_iterate": (st, [i32, P, i64, i64, P, i32, f32, P, P, P, P, P, P, sz, P]),
            "mapi_iterate_host": (st, [i32, P, i64, i64, P, i32, f32, P, P, P, P, P, P, sz, P]),
            "mapi_iterate_host_many": (st, [i32, i32, P, i64, i64, P, i32, f32, P, P, P, P, P, sz, P]),
            "mapi_iterate_sym": (st, [i32, P, i64, i64, P, i32, f32, P, P, P, P, P, P, sz, P]),
            "mapi_iterate_host_many_packed": (st, [i32, i32, P, i64, P, i32, f32, P, P, P, P, P, sz, P]),
            "mapi_iterate_host_many_sym": (st, [i32, i32, P, i64, i64, P, i32, f32, P, P, P, P, P, sz, P]),
            "mapi_pack_upper_host": (st, [P, i64, i64, P, i32]),
            "mapi_iterate_batched": (st, [i32, P, i64, i64, P, i32, i32, f32, P, P, P, P, P, sz, P]),
            "mapi_pca_topk": (st, [i32, P, i64, i64, i32, i32, P, P, P, P, P, sz, P]),
            "mapi_csr_prepare": (st, [i64, i64, P, P, f32, P, P, P, sz, P]),
            "mapi_rank_csr": (st, [i64, i64, P, P, P, P, P, i32, f32, P, P, P, P, P, sz, P]),
            "mapi_rank_csr_shard_begin": (st, [i64, i64, i64, P, P, P, P, P, sz, P]),
            "mapi_rank_csr_shard_rows": (st, [i64, i64, i64, i64, P, P, i32, ctypes.POINTER(ctypes.c_void_p), P, sz,
                                              P]),
            "mapi_rank_csr_shard_normalize": (st, [i64, i64, i64, P, P, P, i32, f32, P, P, sz, P]),
            "mapi_rank_csr_shard_finish": (st, [i64, i64, i64, P, P, P, P, P, P, sz, P]),
            "mapi_csr_reorder": (st, [i64, i64, P, P, P, P, P, P, sz, P]),
            "mapi_csr_plan": (st, [i64, i64, P, P, P, sz, ctypes.POINTER(PlanInfo), P, sz, P]),
            "mapi_rank_csr_plan": (st, [i32, P, ctypes.POINTER(PlanInfo), P, P, P, i32, f32, P, P, P, P, P, sz,
                                        P]),
            "mapi_csr_permute": (st, [i64, P, P, P, i32, P]),
            "mapi_workspace_size": (sz, [i32, i64, i64, i32]),
            "mapi_minibatch": (st, [i32, P, i64, i64, i64, P, i32, i32, f32, P, P, P, P, P, P, ctypes.POINTER(i32), P,
                                    sz, P]),
            "mapi_p2p_exchange_bytes": (sz, [i64, i32]),
            "mapi_p2p_alloc": (st, [sz, ctypes.POINTER(ctypes.c_void_p)]),
            "mapi_p2p_free": (st, [P]),
            "mapi_ipc_get_handle": (st, [P, P]),
            "mapi_ipc_open_handle": (st, [P, ctypes.POINTER(ctypes.c_void_p)]),
            "mapi_ipc_close_handle": (st, [P]),
            "mapi_iterate_sharded": (st, [i32, P, i64, i64, i64, i64, P, i32, f32, i32, i32, P, ctypes.c_uint64,
                                          ctypes.c_uint64, i32, P, P, P, P, P, P, P, sz, P]),
            "mapi_iterate_sym_sharded": (st, [i32, P, i64, i64, i64, i64, P, i32, f32, i32, i32, P,
                                              ctypes.c_uint64, ctypes.c_uint64, i32, P, P, P, P, P, P, P, sz, P]),
            "mapi_sym_shard_rows": (st, [i64, i32, i32, P, P, P, P]),
            "mapi_sym_shard_valid": (st, [i64, i32, i32, i64, P]),
            "mapi_status_string": (ctypes.c_char_p, [st]),
            "mapi_last_error_message": (ctypes.c_char_p, []),
            "mapi_launch_count": (ctypes.c_uint64, []),
            "mapi_set_profiling": (None, [i32]),
            "mapi_last_kernel_ms": (f32, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


# ---------------------------------------------------------------------------------------- helpers


def _torch():
    import torch

    return torch


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream=None) -> Optional[int]:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _check(st: int, iters_done: Optional[int] = None):
    if st != 0:
        msg = load().mapi_last_error_message().decode(errors="replace")
        raise MapiError(st, msg, iters_done)


def _need(t, name, dtype, shape=None, device=True):
    torch = _torch()
    if t is None:
        raise ValueError(f"{name} is required")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if device and not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    del torch


def _matrix(A, name="A"):
    torch = _torch()
    _need(A, name, torch.float32)
    if A.dim() != 2 or A.stride(1) != 1:
        raise ValueError(f"{name} must be a 2-D row-major (stride(1) == 1) fp32 CUDA tensor")
    return A.shape[0], A.shape[1], A.stride(0)


def workspace_size(op: int, n: int, nnz: int = 0, k: int = 0) -> int:
    return int(load().mapi_workspace_size(op, n, nnz, k))


def _workspace(op, n, nnz=0, k=0, device=None, ws=None):
    torch = _torch()
    need = workspace_size(op, n, nnz, k)
    if ws is not None:
        if ws.numel() * ws.element_size() < need:
            raise ValueError(f"workspace too small: {ws.numel() * ws.element_size()} < {need}")
        return ws, need
    return torch.empty(max(need, 256), dtype=torch.uint8, device=device), need


def launch_count() -> int:
    return int(load().mapi_launch_count())


def set_profiling(on: bool) -> None:
    load().mapi_set_profiling(1 if on else 0)


def last_kernel_ms() -> float:
    return float(load().mapi_last_kernel_ms())


# ---------------------------------------------------------------------------------------- API


def mavp_matvec(A, x, y=None, op: int = MIN1, stream=None):
    """y = A (op) x  (matrix extension of Eq. 3/4); asynchronous on `stream`."""
    torch = _torch()
    n_rows, n_cols, lda = _matrix(A)
    _need(x, "x", torch.float32, (n_cols,))
    if y is None:
        y = torch.empty(n_rows, dtype=torch.float32, device=A.device)
    _need(y, "y", torch.float32, (n_rows,))
    _check(load().mapi_mavp_matvec(op, _ptr(A), n_rows, n_cols, lda, _ptr(x), _ptr(y), _stream(stream)))
    return y


def mavp_matmat(A, B, divisor: float = 1.0, C=None, op: int = MIN1, stream=None):
    """C[i][j] = (row_i(A) (op) row_j(B)) / divisor — matrix extension; asynchronous."""
    torch = _torch()
    m, K, lda = _matrix(A, "A")
    p, K2, ldb = _matrix(B, "B")
    if K != K2:
        raise ValueError(f"dimension mismatch: A is {m}x{K}, B is {p}x{K2}")
    if C is None:
        C = torch.empty(m, p, dtype=torch.float32, device=A.device)
    _need(C, "C", torch.float32)
    if C.dim() != 2 or tuple(C.shape) != (m, p) or (C.numel() and C.stride(1) != 1):
        raise ValueError(f"C must be a row-major ({m}, {p}) fp32 tensor")
    _check(load().mapi_mavp_matmat(op, _ptr(A), m, K, lda, _ptr(B), p, ldb, float(divisor), _ptr(C),
                                   C.stride(0) if C.numel() else p, _stream(stream)))
    return C


def min_covariance(V, divisor=None, op: int = MIN1, stream=None):
    """Min-covariance (1/d) V (+) V^T of mean-removed samples V (pixels x N) (Eq. 5):
    d = N - 1 by default as in Alg. 2 step 4."""
    d = (V.shape[1] - 1) if divisor is None else divisor
    return mavp_matmat(V, V, float(d), op=op, stream=stream)


def normalize(y, w, s_out=None, delta_out=None, status_out=None, op: int = MIN1, stream=None):
    """One Algorithm 1 normalisation on a full y: w <- y / ||y|| (l1; l2 for DOT), delta."""
    torch = _torch()
    _need(y, "y", torch.float32)
    _need(w, "w", torch.float32, tuple(y.shape))
    _check(load().mapi_normalize(op, _ptr(y), y.numel(), _ptr(w), _ptr(s_out), _ptr(delta_out), _ptr(status_out),
                                 _stream(stream)))


def center_rows(V, Vc=None, stream=None):
    """Alg. 2 step 3: m = mean over the columns of V (pixels x N), Vc = V - m."""
    torch = _torch()
    M, N, ldv = _matrix(V, "V")
    Vc = torch.empty_like(V) if Vc is None else Vc
    mean = torch.empty(M, dtype=torch.float32, device=V.device)
    _check(load().mapi_center_rows(_ptr(V), M, N, ldv, _ptr(Vc), Vc.stride(0), _ptr(mean), _stream(stream)))
    return Vc, mean


def mavp_deflate(C, w, op: int = MIN1, D=None, ws=None, stream=None):
    """Alg. 2 step 6: D = C - (w (op) w^T) C (regular product; exact O(M^2) evaluation)."""
    torch = _torch()
    M, M2, ldc = _matrix(C, "C")
    if M != M2:
        raise ValueError(f"C must be square, got {tuple(C.shape)}")
    _need(w, "w", torch.float32, (M,))
    D = torch.empty_like(C) if D is None else D
    ws, need = _workspace(WS_MAVP_DEFLATE, M, device=C.device, ws=ws)
    _check(load().mapi_mavp_deflate(op, _ptr(C), M, ldc, _ptr(w), _ptr(D), D.stride(0), _ptr(ws), need,
                                    _stream(stream)))
    return D


def mavp_reconstruct(W, V, op: int = MIN1, Vhat=None, ws=None, stream=None):
    """Alg. 2 steps 3 + 8: v_hat_j = (W (op) W^T)(v_j - m) + m for the columns of V."""
    torch = _torch()
    M, r, ldw = _matrix(W, "W")
    M2, N, ldv = _matrix(V, "V")
    if M != M2:
        raise ValueError(f"dimension mismatch: W has {M} rows, V has {M2}")
    Vhat = torch.empty_like(V) if Vhat is None else Vhat
    mean = torch.empty(M, dtype=torch.float32, device=V.device)
    ws, need = _workspace(WS_RECONSTRUCT, M, N, r, device=V.device, ws=ws)
    _check(load().mapi_mavp_reconstruct(op, _ptr(W), M, r, ldw, _ptr(V), N, ldv, _ptr(Vhat), Vhat.stride(0),
                                        _ptr(mean), _ptr(ws), need, _stream(stream)))
    return Vhat, mean


@dataclass
class IterResult:
    w: object            # l1-unit final iterate (torch / numpy)
    w_l2: object         # l2 copy or None
    norms: object        # s_t = ||A (+) w_t||_1, t < iters_done
    deltas: object       # ||w_{t+1} - w_t||_1
    iters_done: int


def iterate(A, b0, iters: int, tol: float = 0.0, op: int = MIN1, want_l2: bool = True,
            want_trace: bool = True, ws=None, out=None, stream=None) -> IterResult:
    """MAPI, Eq.(8) / Algorithm 1 on device tensors; synchronises the stream."""
    torch = _torch()
    n, n2, lda = _matrix(A)
    if n != n2:
        raise ValueError(f"A must be square, got {tuple(A.shape)}")
    _need(b0, "b0", torch.float32, (n,))
    dev = A.device
    w = out if out is not None else torch.empty(n, dtype=torch.float32, device=dev)
    wl2 = torch.empty(n, dtype=torch.float32, device=dev) if want_l2 else None
    norms = torch.zeros(iters, dtype=torch.float32, device=dev) if want_trace else None
    deltas = torch.zeros(iters, dtype=torch.float32, device=dev) if want_trace else None
    ws, need = _workspace(WS_ITERATE, n, device=dev, ws=ws)
    done = ctypes.c_int32(0)
    st = load().mapi_iterate(op, _ptr(A), n, lda, _ptr(b0), int(iters), float(tol), _ptr(w), _ptr(wl2),
                             _ptr(norms), _ptr(deltas), ctypes.byref(done), _ptr(ws), need,
                             _stream(stream))
    _check(st, done.value)
    k = done.value
    return IterResult(w, wl2, None if norms is None else norms[:k], None if deltas is None else deltas[:k], k)


def iterate_sym(A, b0, iters: int, tol: float = 0.0, op: int = MIN1, want_l2: bool = True,
                want_trace: bool = True, ws=None, out=None, stream=None) -> IterResult:
    """MAPI on a SYMMETRIC device matrix reading only its upper triangle (mapi_iterate_sym, K2s); the
    caller declares symmetry.  Synchronises the stream."""
    torch = _torch()
    n, n2, lda = _matrix(A)
    if n != n2:
        raise ValueError(f"A must be square, got {tuple(A.shape)}")
    _need(b0, "b0", torch.float32, (n,))
    dev = A.device
    w = out if out is not None else torch.empty(n, dtype=torch.float32, device=dev)
    wl2 = torch.empty(n, dtype=torch.float32, device=dev) if want_l2 else None
    norms = torch.zeros(iters, dtype=torch.float32, device=dev) if want_trace else None
    deltas = torch.zeros(iters, dtype=torch.float32, device=dev) if want_trace else None
    ws, need = _workspace(WS_ITERATE_SYM, n, device=dev, ws=ws)
    done = ctypes.c_int32(0)
    st = load().mapi_iterate_sym(op, _ptr(A), n, lda, _ptr(b0), int(iters), float(tol), _ptr(w), _ptr(wl2),
                                 _ptr(norms), _ptr(deltas), ctypes.byref(done), _ptr(ws), need,
                                 _stream(stream))
    _check(st, done.value)
    k = done.value
    return IterResult(w, wl2, None if norms is None else norms[:k], None if deltas is None else deltas[:k], k)


def iterate_host(A_host, b0_host, iters: int, tol: float = 0.0, op: int = MIN1, ws=None,
                 out=None, norms=None, deltas=None, stream=None) -> IterResult:
    """MAPI end-to-end from HOST buffers (torch CPU tensors, ideally pinned): the call copies A, b0
    to the device workspace, iterates, and copies w / trace back.  Synchronises the stream."""
    torch = _torch()
    if A_host.is_cuda or b0_host.is_cuda:
        raise ValueError("iterate_host takes host (CPU) tensors")
    if A_host.dtype != torch.float32 or A_host.dim() != 2 or A_host.stride(1) != 1:
        raise ValueError("A_host must be a 2-D row-major fp32 CPU tensor")
    n, lda = A_host.shape[0], A_host.stride(0)
    w = out if out is not None else torch.empty(n, dtype=torch.float32)
    norms = norms if norms is not None else torch.zeros(iters, dtype=torch.float32)
    deltas = deltas if deltas is not None else torch.zeros(iters, dtype=torch.float32)
    ws, need = _workspace(WS_ITERATE_HOST, n, lda, iters, device=torch.device("cuda"), ws=ws)
    done = ctypes.c_int32(0)
    st = load().mapi_iterate_host(op, _ptr(A_host), n, lda, _ptr(b0_host), int(iters), float(tol), _ptr(w),
                                  None, _ptr(norms), _ptr(deltas), ctypes.byref(done), _ptr(ws), need,
                                  _stream(stream))
    _check(st, done.value)
    k = done.value
    return IterResult(w, None, norms[:k], deltas[:k], k)


def iterate_host_many(As, b0s, iters: int, tol: float = 0.0, op: int = MIN1, ws=None, outs=None,
                      want_trace: bool = True, stream=None) -> list:
    """`len(As)` independent MAPI problems from HOST buffers (pinned CPU tensors), pipelined: the next
    problem's host->device copy overlaps the current one's iterations (mapi_iterate_host_many).  All
    problems share n / lda.  Returns one IterResult per problem; synchronises the stream."""
    torch = _torch()
    count = len(As)
    if count < 1 or len(b0s) != count:
        raise ValueError("need >= 1 problem and one b0 per problem")
    n, lda = As[0].shape[0], As[0].stride(0)
    for A, b in zip(As, b0s):
        if A.is_cuda or b.is_cuda or A.dtype != torch.float32 or A.dim() != 2 or A.stride(1) != 1:
            raise ValueError("As must be 2-D row-major fp32 CPU tensors (pinned for overlap)")
        if A.shape[0] != n or A.stride(0) != lda or b.numel() != n:
            raise ValueError("every problem must have the same n and lda")
    outs = outs if outs is not None else [torch.empty(n, dtype=torch.float32) for _ in range(count)]
    pin = torch.cuda.is_available()
    norms = [torch.zeros(iters, dtype=torch.float32, pin_memory=pin) for _ in range(count)] if want_trace else None
    deltas = [torch.zeros(iters, dtype=torch.float32, pin_memory=pin) for _ in range(count)] if want_trace else None
    lib = load()
    need = int(lib.mapi_workspace_size(WS_ITERATE_HOST_MANY, n, lda, iters)) + 8 * max(0, count - 2)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    arr = lambda ts: (ctypes.c_void_p * count)(*[t.data_ptr() for t in ts])  # noqa: E731
    done = (ctypes.c_int32 * count)()
    st = lib.mapi_iterate_host_many(op, count, arr(As), n, lda, arr(b0s), int(iters), float(tol), arr(outs),
                                    arr(norms) if norms else None, arr(deltas) if deltas else None, done,
                                    _ptr(ws), ws.numel(), _stream(stream))
    _check(st)
    res = []
    for i in range(count):
        k = done[i]
        res.append(IterResult(outs[i], None, norms[i][:k] if norms else None, deltas[i][:k] if deltas else None, k))
    return res


def pack_upper(A, out=None, threads: int = 0):
    """Host-side input preparation for iterate_host_many_packed: the upper triangle of a symmetric n x n
    fp32 CPU matrix in packed row-major order (row j = A[j, j:], LAPACK "packed" layout), n(n+1)/2 floats,
    copied by `threads` native host threads (mapi_pack_upper_host; 0 = all).  Pure data movement (no
    arithmetic); `out` may be a pinned 1-D fp32 tensor to fill."""
    torch = _torch()
    A = torch.as_tensor(A)
    if A.dim() != 2 or A.shape[0] != A.shape[1] or A.dtype != torch.float32 or A.is_cuda or A.stride(1) != 1:
        raise ValueError("A must be a square row-major fp32 CPU matrix")
    n = A.shape[0]
    out = out if out is not None else torch.empty(n * (n + 1) // 2, dtype=torch.float32)
    if out.numel() != n * (n + 1) // 2 or not out.is_contiguous():
        raise ValueError("out must be a contiguous tensor of n(n+1)/2 floats")
    _check(load().mapi_pack_upper_host(A.data_ptr(), n, A.stride(0), out.data_ptr(), int(threads)))
    return out


def iterate_host_many_sym(As, b0s, iters: int, tol: float = 0.0, op: int = MIN1, ws=None, outs=None,
                          want_trace: bool = True, stream=None) -> list:
    """iterate_host_many for SYMMETRIC matrices given as full pinned host matrices: only the upper-triangle
    block rows cross PCIe (mapi_iterate_host_many_sym: one 2-D copy per 128-row block), K2s iterates on them.
    Returns one IterResult per problem; synchronises the stream."""
    torch = _torch()
    count = len(As)
    if count < 1 or len(b0s) != count:
        raise ValueError("need >= 1 problem and one b0 per problem")
    n = As[0].shape[0]
    for A, b in zip(As, b0s):
        if A.is_cuda or b.is_cuda or A.dtype != torch.float32 or A.dim() != 2 or A.shape[0] != n or \
                A.stride(1) != 1 or A.stride(0) != As[0].stride(0):
            raise ValueError("As must be n x lda row-major fp32 CPU tensors with one lda (pinned for overlap)")
    lda = As[0].stride(0)
    outs = outs if outs is not None else [torch.empty(n, dtype=torch.float32) for _ in range(count)]
    pin = torch.cuda.is_available()
    norms = [torch.zeros(iters, dtype=torch.float32, pin_memory=pin) for _ in range(count)] if want_trace else None
    deltas = [torch.zeros(iters, dtype=torch.float32, pin_memory=pin) for _ in range(count)] if want_trace else None
    lib = load()
    need = int(lib.mapi_workspace_size(WS_ITERATE_HOST_MANY_SYM, n, 0, iters)) + 8 * max(0, count - 2)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    arr = lambda ts: (ctypes.c_void_p * count)(*[t.data_ptr() for t in ts])  # noqa: E731
    done = (ctypes.c_int32 * count)()
    st = lib.mapi_iterate_host_many_sym(op, count, arr(As), n, lda, arr(b0s), int(iters), float(tol), arr(outs),
                                        arr(norms) if norms else None, arr(deltas) if deltas else None, done,
                                        _ptr(ws), ws.numel(), _stream(stream))
    _check(st)
    res = []
    for i in range(count):
        k = done[i]
        res.append(IterResult(outs[i], None, norms[i][:k] if norms else None, deltas[i][:k] if deltas else None, k))
    return res


def iterate_host_many_packed(Aps, n: int, b0s, iters: int, tol: float = 0.0, op: int = MIN1, ws=None, outs=None,
                             want_trace: bool = True, stream=None) -> list:
    """iterate_host_many for symmetric matrices sent as packed upper triangles (pack_upper): half the
    host->device bytes; the device rebuilds each full matrix bitwise before iterating
    (mapi_iterate_host_many_packed).  Returns one IterResult per problem; synchronises the stream."""
    torch = _torch()
    count = len(Aps)
    if count < 1 or len(b0s) != count:
        raise ValueError("need >= 1 problem and one b0 per problem")
    for Ap, b in zip(Aps, b0s):
        if Ap.is_cuda or b.is_cuda or Ap.dtype != torch.float32 or not Ap.is_contiguous():
            raise ValueError("Aps must be contiguous fp32 CPU tensors (pinned for overlap)")
        if Ap.numel() != n * (n + 1) // 2 or b.numel() != n:
            raise ValueError(f"each packed matrix must hold n(n+1)/2 = {n * (n + 1) // 2} floats and b0 n floats")
    outs = outs if outs is not None else [torch.empty(n, dtype=torch.float32) for _ in range(count)]
    pin = torch.cuda.is_available()
    norms = [torch.zeros(iters, dtype=torch.float32, pin_memory=pin) for _ in range(count)] if want_trace else None
    deltas = [torch.zeros(iters, dtype=torch.float32, pin_memory=pin) for _ in range(count)] if want_trace else None
    lib = load()
    need = int(lib.mapi_workspace_size(WS_ITERATE_HOST_MANY_PACKED, n, 0, iters)) + 8 * max(0, count - 2)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    arr = lambda ts: (ctypes.c_void_p * count)(*[t.data_ptr() for t in ts])  # noqa: E731
    done = (ctypes.c_int32 * count)()
    st = lib.mapi_iterate_host_many_packed(op, count, arr(Aps), n, arr(b0s), int(iters), float(tol), arr(outs),
                                           arr(norms) if norms else None, arr(deltas) if deltas else None, done,
                                           _ptr(ws), ws.numel(), _stream(stream))
    _check(st)
    res = []
    for i in range(count):
        k = done[i]
        res.append(IterResult(outs[i], None, norms[i][:k] if norms else None, deltas[i][:k] if deltas else None, k))
    return res


@dataclass
class BatchedResult:
    W: object            # k x n, l1-unit rows
    norms: object        # iters x k
    deltas: object       # iters x k
    iters_done: list


def iterate_batched(A, B0, iters: int, tol: float = 0.0, op: int = MIN1, ws=None,
                    stream=None) -> BatchedResult:
    """k independent MAPI runs on one A (matrix extension P:69-70); synchronises the stream."""
    torch = _torch()
    n, n2, lda = _matrix(A)
    if n != n2:
        raise ValueError(f"A must be square, got {tuple(A.shape)}")
    _need(B0, "B0", torch.float32)
    if B0.dim() != 2 or B0.shape[1] != n or not B0.is_contiguous():
        raise ValueError(f"B0 must be a contiguous (k, {n}) tensor")
    k = B0.shape[0]
    dev = A.device
    W = torch.empty_like(B0)
    norms = torch.zeros(iters, k, dtype=torch.float32, device=dev)
    deltas = torch.zeros(iters, k, dtype=torch.float32, device=dev)
    ws, need = _workspace(WS_ITERATE_BATCHED, n, 0, k, device=dev, ws=ws)
    done = (ctypes.c_int32 * k)()
    st = load().mapi_iterate_batched(op, _ptr(A), n, lda, _ptr(B0), k, int(iters), float(tol), _ptr(W),
                                     _ptr(norms), _ptr(deltas), done, _ptr(ws), need, _stream(stream))
    _check(st)
    return BatchedResult(W, norms, deltas, list(done))


@dataclass
class PcaResult:
    P: object            # k x n, l2-unit rows
    norms: object        # k x iters
    deltas: object       # k x iters


def pca_topk(C, k: int, iters: int, b0, op: int = MIN1, ws=None, stream=None) -> PcaResult:
    """Top-k principal vectors by MAPI with L2 deflation; synchronises the stream."""
    torch = _torch()
    n, n2, ldc = _matrix(C, "C")
    if n != n2:
        raise ValueError(f"C must be square, got {tuple(C.shape)}")
    _need(b0, "b0", torch.float32, (n,))
    dev = C.device
    P = torch.empty(k, n, dtype=torch.float32, device=dev)
    norms = torch.zeros(k, iters, dtype=torch.float32, device=dev)
    deltas = torch.zeros(k, iters, dtype=torch.float32, device=dev)
    ws, need = _workspace(WS_PCA_TOPK, n, 0, k, device=dev, ws=ws)
    st = load().mapi_pca_topk(op, _ptr(C), n, ldc, int(k), int(iters), _ptr(b0), _ptr(P), _ptr(norms),
                              _ptr(deltas), _ptr(ws), need, _stream(stream))
    _check(st)
    return PcaResult(P, norms, deltas)


def csr_prepare(n: int, row_ptr, col_idx, alpha: float = 0.85, ws=None, stream=None):
    """Per-column cap_j = alpha/outdeg(j) and bg_j of the Google matrix (Eq. 13)."""
    torch = _torch()
    _need(row_ptr, "row_ptr", torch.int32, (n + 1,))
    _need(col_idx, "col_idx", torch.int32)
    nnz = col_idx.numel()
    dev = row_ptr.device
    cap = torch.empty(n, dtype=torch.float32, device=dev)
    bg = torch.empty(n, dtype=torch.float32, device=dev)
    ws, need = _workspace(WS_CSR_PREPARE, n, nnz, device=dev, ws=ws)
    _check(load().mapi_csr_prepare(n, nnz, _ptr(row_ptr), _ptr(col_idx) if nnz else None, float(alpha),
                                   _ptr(cap), _ptr(bg), _ptr(ws), need, _stream(stream)))
    return cap, bg


def rank_csr(n: int, row_ptr, col_idx, cap, bg, b0, max_iters: int = 200, tol: float = 1e-7,
             want_l2: bool = True, ws=None, stream=None) -> IterResult:
    """MAPI ranking on G = alpha M + (1-alpha)/n 1 (Eq. 13); synchronises the stream."""
    torch = _torch()
    _need(row_ptr, "row_ptr", torch.int32, (n + 1,))
    _need(col_idx, "col_idx", torch.int32)
    for name, t in (("cap", cap), ("bg", bg), ("b0", b0)):
        _need(t, name, torch.float32, (n,))
    nnz = col_idx.numel()
    dev = row_ptr.device
    w = torch.empty(n, dtype=torch.float32, device=dev)
    wl2 = torch.empty(n, dtype=torch.float32, device=dev) if want_l2 else None
    deltas = torch.zeros(max_iters, dtype=torch.float32, device=dev)
    ws, need = _workspace(WS_RANK_CSR, n, nnz, device=dev, ws=ws)
    done = ctypes.c_int32(0)
    st = load().mapi_rank_csr(n, nnz, _ptr(row_ptr), _ptr(col_idx) if nnz else None, _ptr(cap), _ptr(bg),
                              _ptr(b0), int(max_iters), float(tol), _ptr(w), _ptr(wl2), _ptr(deltas),
                              ctypes.byref(done), _ptr(ws), need, _stream(stream))
    _check(st, done.value)
    k = done.value
    return IterResult(w, wl2, None, deltas[:k], k)

def minibatch(X, batch, beta: float, w0, gram: int = MIN1, want_l2: bool = True, w_prev0=None, ws=None,
              stream=None) -> IterResult:
    """Algorithm 3, mini-batch MAPI with momentum (mapi_minibatch): X N x D fp32 samples, batch
    T x s int32 row indices (the caller's draws), w0 D, w_prev0 the momentum vector of a continued run (None:
    w_{-1} = 0).  norms[t] = ||w_{t+1}||_1 before normalisation; the `deltas` field carries the momentum
    vector after the last step (w_prev, for continuing).  Synchronises the stream."""
    torch = _torch()
    N, D, ldx = _matrix(X, "X")
    _need(batch, "batch", torch.int32)
    if batch.dim() != 2 or not batch.is_contiguous():
        raise ValueError("batch must be a contiguous (T, s) int32 tensor")
    T, s = batch.shape
    _need(w0, "w0", torch.float32, (D,))
    if w_prev0 is not None:
        _need(w_prev0, "w_prev0", torch.float32, (D,))
    dev = X.device
    w = torch.empty(D, dtype=torch.float32, device=dev)
    wl2 = torch.empty(D, dtype=torch.float32, device=dev) if want_l2 else None
    wprev = torch.empty(D, dtype=torch.float32, device=dev)
    norms = torch.zeros(max(T, 1), dtype=torch.float32, device=dev)
    ws, need = _workspace(WS_MINIBATCH, D, s, T, device=dev, ws=ws)
    done = ctypes.c_int32(0)
    st = load().mapi_minibatch(gram, _ptr(X), N, D, ldx, _ptr(batch), int(s), int(T), float(beta), _ptr(w0),
                               _ptr(w_prev0), _ptr(w), _ptr(wl2), _ptr(wprev), _ptr(norms), ctypes.byref(done),
                               _ptr(ws), need, _stream(stream))
    _check(st, done.value)
    k = done.value
    return IterResult(w, wl2, norms[:k], wprev, k)


class PlanInfo(ctypes.Structure):
    """mapi_csr_plan_info (include/mapi.h): sizes of a segmented ranking plan."""
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64), ("nsrc", ctypes.c_int64),
                ("npieces", ctypes.c_int64), ("nwords", ctypes.c_int64), ("nseg", ctypes.c_int32),
                ("grid", ctypes.c_int32), ("nlive", ctypes.c_int64), ("nbatch", ctypes.c_int64),
                ("nunits", ctypes.c_int64)]


@dataclass
class CsrPlan:
    buf: object          # device uint8 tensor holding the plan
    info: PlanInfo


def csr_plan(n: int, row_ptr, col_idx, ws=None, stream=None) -> CsrPlan:
    """One-time segmented layout of the graph for rank_csr_plan (mapi_csr_plan, K3s);
    synchronises the stream."""
    torch = _torch()
    _need(row_ptr, "row_ptr", torch.int32, (n + 1,))
    _need(col_idx, "col_idx", torch.int32)
    nnz = col_idx.numel()
    dev = row_ptr.device
    bytes_ = workspace_size(WS_CSR_PLAN, n, nnz)
    buf = torch.empty(max(bytes_, 256), dtype=torch.uint8, device=dev)
    ws, need = _workspace(WS_CSR_PLAN_BUILD, n, nnz, device=dev, ws=ws)
    info = PlanInfo()
    _check(load().mapi_csr_plan(n, nnz, _ptr(row_ptr), _ptr(col_idx) if nnz else None, _ptr(buf), bytes_,
                                ctypes.byref(info), _ptr(ws), need, _stream(stream)))
    return CsrPlan(buf, info)


def rank_csr_plan(plan: CsrPlan, cap, bg, b0, max_iters: int = 200, tol: float = 1e-7, op: int = MIN1,
                  want_l2: bool = True, ws=None, stream=None) -> IterResult:
    """MAPI (op MIN1/MIN2) or PageRank RPI (op DOT) ranking through a plan (mapi_rank_csr_plan, K3s);
    synchronises the stream."""
    torch = _torch()
    n = plan.info.n
    for name, t in (("cap", cap), ("bg", bg), ("b0", b0)):
        _need(t, name, torch.float32, (n,))
    dev = b0.device
    w = torch.empty(n, dtype=torch.float32, device=dev)
    wl2 = torch.empty(n, dtype=torch.float32, device=dev) if want_l2 else None
    deltas = torch.zeros(max_iters, dtype=torch.float32, device=dev)
    ws, need = _workspace(WS_RANK_CSR_PLAN, n, plan.info.nnz, device=dev, ws=ws)
    done = ctypes.c_int32(0)
    st = load().mapi_rank_csr_plan(op, _ptr(plan.buf), ctypes.byref(plan.info), _ptr(cap), _ptr(bg), _ptr(b0),
                                   int(max_iters), float(tol), _ptr(w), _ptr(wl2), _ptr(deltas),
                                   ctypes.byref(done), _ptr(ws), need, _stream(stream))
    _check(st, done.value)
    k = done.value
    return IterResult(w, wl2, None, deltas[:k], k)


def csr_reorder(n: int, row_ptr, col_idx, ws=None, stream=None):
    """Relabel the graph's nodes by descending out-degree (mapi_csr_reorder): returns (perm, row_ptr',
    col_idx') with perm[old] = new.  Asynchronous."""
    torch = _torch()
    _need(row_ptr, "row_ptr", torch.int32, (n + 1,))
    _need(col_idx, "col_idx", torch.int32)
    nnz = col_idx.numel()
    dev = row_ptr.device
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
    ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)[:nnz]
    ws, need = _workspace(WS_CSR_REORDER, n, device=dev, ws=ws)
    _check(load().mapi_csr_reorder(n, nnz, _ptr(row_ptr), _ptr(col_idx) if nnz else None, _ptr(perm), _ptr(rp),
                                   _ptr(ci) if nnz else None, _ptr(ws), need, _stream(stream)))
    return perm, rp, ci


def csr_permute(perm, x, to_new: bool = True, out=None, stream=None):
    """out[perm[j]] = x[j] (to_new) or out[j] = x[perm[j]] (back to the original ids); asynchronous."""
    torch = _torch()
    n = perm.numel()
    _need(perm, "perm", torch.int32, (n,))
    _need(x, "x", torch.float32, (n,))
    out = out if out is not None else torch.empty_like(x)
    _check(load().mapi_csr_permute(n, _ptr(perm), _ptr(x), _ptr(out), 1 if to_new else 0, _stream(stream)))
    return out

