"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no MAVP, no normalisation, no
deflation, no Google-matrix weights): it only draws the inputs that BASELINE.json's
configs describe, with the recipes fixed in DESIGN.md §"Input recipes":

* ``numpy.random.default_rng(seed)`` (PCG64), fp64 draws, fp64 arithmetic, ONE cast to
  fp32 per stored array;
* covariance-like matrices are formed block-wise and mirrored so that the fp32 result is
  exactly symmetric (the setup product ``X X^T / N`` is the paper's Eq.(2), P:21-25 — input
  preparation, formed once, off the timed path, BASELINE north_star);
* graphs are returned as a destination-major CSR structure (row i lists the sources j of
  the distinct edges j -> i, reading Q10/Q11); per-edge weights are NOT produced here.

The heavy setup product can run through torch on a CUDA device (cuBLAS DGEMM) purely as
input preparation; the draws are always numpy so both sides see the same recipe.
"""
from __future__ import annotations

import hashlib

import numpy as np

__all__ = ["cfg1", "cfg2", "cfg3", "cfg3_rows", "covariance_like_rows", "cfg4", "cfg5", "gnutella_like", "occluded_images", "occluded_copies", "rmat_edges",
           "csr_by_destination", "random_matrix", "random_graph", "digest", "covariance_like"]


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(memoryview(a).cast("B"))
    return h.hexdigest()


# ----------------------------------------------------------------------------------------
# dense covariance-like matrices


def _sym_product_blocks(F, scale, diag, out, block, device):
    """out[:] = fp32( F F^T * scale + diag(diag) ), block upper triangle mirrored (exact symmetry).

    ``out`` is a numpy float32 array (device None) or a torch float32 tensor on ``device``.
    """
    n = F.shape[0]
    if device is None:
        Fd = F
        for r0 in range(0, n, block):
            r1 = min(n, r0 + block)
            for c0 in range(r0, n, block):
                c1 = min(n, c0 + block)
                M = (Fd[r0:r1] @ Fd[c0:c1].T) * scale
                if r0 == c0:
                    M[np.arange(r1 - r0), np.arange(r1 - r0)] += diag[r0:r1]
                    M = np.triu(M) + np.triu(M, 1).T
                M32 = M.astype(np.float32)
                out[r0:r1, c0:c1] = M32
                if c0 != r0:
                    out[c0:c1, r0:r1] = M32.T
        return out
    import torch

    Fd = torch.from_numpy(F).to(device)
    dd = torch.from_numpy(np.asarray(diag, dtype=np.float64)).to(device)
    for r0 in range(0, n, block):
        r1 = min(n, r0 + block)
        for c0 in range(r0, n, block):
            c1 = min(n, c0 + block)
            M = (Fd[r0:r1] @ Fd[c0:c1].T) * scale
            if r0 == c0:
                idx = torch.arange(r1 - r0, device=device)
                M[idx, idx] += dd[r0:r1]
                M = torch.triu(M) + torch.triu(M, 1).T
            M32 = M.to(torch.float32)
            out[r0:r1, c0:c1] = M32
            if c0 != r0:
                out[c0:c1, r0:r1] = M32.T
        del M
    return out


def covariance_like(F, scale, diag=None, device=None, block=4096):
    """fp32 symmetric ``F F^T * scale + diag(diag)`` (numpy out, or torch on ``device``)."""
    n = F.shape[0]
    if diag is None:
        diag = np.zeros(n)
    if device is None:
        out = np.empty((n, n), np.float32)
    else:
        import torch

        out = torch.empty((n, n), dtype=torch.float32, device=device)
    return _sym_product_blocks(np.ascontiguousarray(F, dtype=np.float64), scale,
                               np.asarray(diag, np.float64), out, block, device)


def covariance_like_rows(F, scale, diag, row0, row1, device=None, block=4096):
    """Rows [row0, row1) of covariance_like(F, scale, diag, device, block), computed with the same block
    convention (upper-triangle blocks as F_bi F_bj^T, lower ones as their transposes), so every rank of a
    row-sharded run generates exactly its slice of the same matrix.  row0 must be a multiple of block."""
    n = F.shape[0]
    if row0 % block != 0:
        raise ValueError("row0 must be a multiple of the block size")
    F = np.ascontiguousarray(F, dtype=np.float64)
    diag = np.asarray(diag, np.float64)
    if device is None:
        out = np.empty((row1 - row0, n), np.float32)
        mm = lambda a, b: a @ b.T  # noqa: E731
        Fd = F
    else:
        import torch

        out = torch.empty((row1 - row0, n), dtype=torch.float32, device=device)
        Fd = torch.from_numpy(F).to(device)
        mm = lambda a, b: a @ b.T  # noqa: E731
    for r0 in range(row0, row1, block):
        r1 = min(row1, r0 + block)
        for c0 in range(0, n, block):
            c1 = min(n, c0 + block)
            if c0 >= r0:
                M = mm(Fd[r0:r1], Fd[c0:c1]) * scale
                if c0 == r0:
                    idx = np.arange(r1 - r0)
                    if device is None:
                        M[idx, idx] += diag[r0:r1]
                        M = np.triu(M) + np.triu(M, 1).T
                    else:
                        import torch

                        ti = torch.arange(r1 - r0, device=device)
                        M[ti, ti] += torch.from_numpy(diag[r0:r1]).to(device)
                        M = torch.triu(M) + torch.triu(M, 1).T
                blk = M.astype(np.float32) if device is None else M.to(torch.float32)
            else:  # lower block: transpose of the (c, r) upper block, as covariance_like mirrors it
                M = mm(Fd[c0:c1], Fd[r0:r1]) * scale
                blk = (M.astype(np.float32) if device is None else M.to(torch.float32)).T
            out[r0 - row0:r1 - row0, c0:c1] = blk
    return out


def cfg3_rows(row0, row1, device=None, n=32768, rank=512):
    """Rows [row0, row1) of cfg3's A (row-sharded multi-GPU runs)."""
    r = np.random.default_rng(2)
    G = r.standard_normal((n, rank))
    z = r.standard_normal(n)
    A = covariance_like_rows(G, 1.0 / n, 10.0 * np.abs(z), row0, row1, device=device)
    b0 = np.full(n, 1.0 / np.sqrt(n), dtype=np.float32)
    return {"name": "cfg3", "A": A, "b0": b0, "iters": 100, "tol": 0.0, "row0": row0, "row1": row1}


def cfg1():
    """BJ configs[0]: X 256x1024 N(0,1) seed 0, row-centred, cast fp32; C = X X^T / 1024
    (fp64 product of the fp32 X, one fp32 cast); b0 = ones/sqrt(256); 50 iterations."""
    r = np.random.default_rng(0)
    X = r.standard_normal((256, 1024))
    X = X - X.mean(axis=1, keepdims=True)
    X32 = X.astype(np.float32).astype(np.float64)
    C = covariance_like(X32, 1.0 / 1024)
    b0 = np.full(256, 1.0 / 16.0, dtype=np.float32)
    return {"name": "cfg1", "A": C, "b0": b0, "iters": 50, "tol": 0.0}


def cfg2(device=None):
    """BJ configs[1] (reading Q15): X 4096x8192 U[0,1) seed 1; Bernoulli(0.05) mask replaced by
    +-10 (equal probability); rows centred over 8192 columns; C = X X^T / 8192 -> fp32;
    b0 = ones/sqrt(4096); top-8 vectors, 100 iterations each."""
    r = np.random.default_rng(1)
    X = r.uniform(0.0, 1.0, (4096, 8192))
    m = r.random(X.shape) < 0.05
    X[m] = 10.0 * r.choice(np.array([-1.0, 1.0]), int(m.sum()))
    X = X - X.mean(axis=1, keepdims=True)
    C = covariance_like(X, 1.0 / 8192, device=device)
    b0 = np.full(4096, 1.0 / 64.0, dtype=np.float32)
    return {"name": "cfg2", "A": C, "b0": b0, "k": 8, "iters": 100, "tol": 0.0}


def _gram_diag(n, rank, seed, device):
    r = np.random.default_rng(seed)
    G = r.standard_normal((n, rank))
    z = r.standard_normal(n)
    A = covariance_like(G, 1.0 / n, 10.0 * np.abs(z), device=device)
    return r, A


def cfg3(device=None, n=32768, rank=512):
    """BJ configs[2]: A = G G^T / n + diag(10|z|), G n x 512 N(0,1), z N(0,1), seed 2, fp32
    (4 GiB at n = 32768); b0 = ones/sqrt(n); 100 iterations."""
    _, A = _gram_diag(n, rank, 2, device)
    b0 = np.full(n, 1.0 / np.sqrt(n), dtype=np.float32)
    return {"name": "cfg3", "A": A, "b0": b0, "iters": 100, "tol": 0.0}


def cfg4(device=None, n=16384, rank=256, k=64):
    """BJ configs[3] (reading Q14): same construction at n = 16384, rank 256, seed 3; the k = 64
    starting vectors continue the seed-3 stream: N(0,1) rows, each l2-normalised; 100 iterations."""
    r, A = _gram_diag(n, rank, 3, device)
    B0 = r.standard_normal((k, n))
    B0 = B0 / np.sqrt(np.sum(B0 * B0, axis=1, keepdims=True))
    return {"name": "cfg4", "A": A, "B0": B0.astype(np.float32), "iters": 100, "tol": 0.0}


# ----------------------------------------------------------------------------------------
# graphs


def rmat_edges(scale, n_edges, a=0.57, b=0.19, c=0.19, seed=4):
    """R-MAT edge list (reading Q12): per edge and per level (MSB first) one U[0,1) draw u;
    quadrant a (src 0, dst 0) if u < a; b (0, 1) if u < a+b; c (1, 0) if u < a+b+c; else d (1, 1).
    Drawn level-major (one n_edges-vector per level).  Returns (src, dst) int64."""
    r = np.random.default_rng(seed)
    src = np.zeros(n_edges, np.int64)
    dst = np.zeros(n_edges, np.int64)
    t_ab, t_abc = a + b, a + b + c
    for _ in range(scale):
        u = r.random(n_edges)
        sbit = u >= t_ab
        dbit = ((u >= a) & (u < t_ab)) | (u >= t_abc)
        src <<= 1
        dst <<= 1
        src |= sbit
        dst |= dbit
        del u, sbit, dbit
    return src, dst


def csr_by_destination(n, src, dst):
    """Distinct edges (duplicates collapsed, self-loops kept, reading Q11) as CSR by destination:
    row i = sorted sources j of edges j -> i.  row_ptr int64 (n+1), col_idx int32."""
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    key = np.unique(dst * np.int64(n) + src)
    d = key // n
    s = (key - d * n).astype(np.int32)
    counts = np.bincount(d, minlength=n)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return row_ptr, s


def cfg5(scale=22, edge_factor=16, seed=4):
    """BJ configs[4]: R-MAT 2^22 nodes, 2^26 edges (a,b,c,d = .57,.19,.19,.05, seed 4), distinct
    edges, destination-major CSR; b0 = 1/n; alpha = 0.85; tol 1e-7 or 200 iterations."""
    n = 1 << scale
    src, dst = rmat_edges(scale, n * edge_factor, seed=seed)
    row_ptr, col_idx = csr_by_destination(n, src, dst)
    del src, dst
    b0 = np.full(n, 1.0 / n, dtype=np.float32)
    return {"name": "cfg5", "n": n, "row_ptr": row_ptr, "col_idx": col_idx, "b0": b0,
            "alpha": 0.85, "max_iters": 200, "tol": 1e-7}


def gnutella_like(n=6301, n_edges=20777, seed=5):
    """Gnutella08-shaped stand-in (P:326 sizes): n nodes, n_edges distinct uniformly
    random directed edges, seed 5.  A light-tailed stand-in, not the SNAP dataset."""
    r = np.random.default_rng(seed)
    seen = set()
    out = []
    while len(out) < n_edges:
        cand = r.integers(0, n, size=(2 * n_edges, 2))
        for s, d in cand:
            k = int(s) * n + int(d)
            if k not in seen:
                seen.add(k)
                out.append((int(s), int(d)))
                if len(out) == n_edges:
                    break
    e = np.array(out, np.int64)
    row_ptr, col_idx = csr_by_destination(n, e[:, 0], e[:, 1])
    b0 = np.full(n, 1.0 / n, dtype=np.float32)
    return {"name": "gnutella_like", "n": n, "row_ptr": row_ptr, "col_idx": col_idx, "b0": b0,
            "edges": e, "alpha": 0.85, "max_iters": 200, "tol": 1e-7}


def random_graph(n, p_edge, seed, n_dangling=0):
    """Erdos-Renyi-style digraph with `n_dangling` forced dangling nodes (outdeg 0).
    Returns (edges int64 (E,2) as (src, dst), row_ptr, col_idx)."""
    r = np.random.default_rng(seed)
    M = r.random((n, n)) < p_edge
    if n_dangling:
        dang = r.choice(n, size=n_dangling, replace=False)
        M[dang, :] = False
    src, dst = np.nonzero(M)
    row_ptr, col_idx = csr_by_destination(n, src, dst)
    return np.stack([src, dst], 1).astype(np.int64), row_ptr, col_idx


def occluded_copies(D=128, N=10, seed=6, tiles=3, tile=32):
    """Stand-in for the paper's image-reconstruction input (Alg. 2 steps 1-2): a smooth
    synthetic D x D "image" with pixels in [0, 1] (sum of random low-frequency cosines, min-max
    scaled) and N copies, each with `tiles` of the (D/tile)^2 tiles replaced by i.i.d. U[0,1] noise.
    Returns (V raw, D^2 x N fp32, the images as columns; the clean image, D x D fp64).
    Not the paper's images (unpublished): same shape, value range and corruption model."""
    r = np.random.default_rng(seed)
    yy, xx = np.meshgrid(np.arange(D) / D, np.arange(D) / D, indexing="ij")
    img = np.zeros((D, D))
    for _ in range(6):
        fx, fy = r.integers(1, 5, size=2)
        img += r.uniform(0.3, 1.0) * np.cos(2 * np.pi * (fx * xx + fy * yy) + r.uniform(0, 2 * np.pi))
    img = (img - img.min()) / (img.max() - img.min())
    per = D // tile
    V = np.empty((D * D, N))
    for i in range(N):
        x = img.copy()
        for t in r.choice(per * per, size=tiles, replace=False):
            ty, tx = divmod(int(t), per)
            x[ty * tile:(ty + 1) * tile, tx * tile:(tx + 1) * tile] = r.random((tile, tile))
        V[:, i] = x.reshape(-1)
    return V.astype(np.float32), img


def occluded_images(D=128, N=10, seed=6, tiles=3, tile=32):
    """occluded_copies after the mean removal of Alg. 2 step 3: (V centred fp32, clean image)."""
    V, img = occluded_copies(D, N, seed, tiles, tile)
    V64 = V.astype(np.float64)
    return (V64 - V64.mean(axis=1, keepdims=True)).astype(np.float32), img


# ----------------------------------------------------------------------------------------
# small generic inputs for kernel tests


def random_matrix(n_rows, n_cols, seed, lda=None, kind="normal"):
    """Seeded fp32 matrix with leading dimension lda (>= n_cols; padding filled with NaN so a
    kernel that reads past n_cols is caught).  kind:
      normal  N(0,1)
      mixed   N(0,1) with injected +-0, rows of zeros, huge (1e30) and tiny (1e-30) magnitudes
      uniform U[0,1)
    Returns (M, lda) where M is the full (n_rows, lda) fp32 buffer."""
    r = np.random.default_rng(seed)
    lda = n_cols if lda is None else lda
    M = np.full((n_rows, lda), np.nan, dtype=np.float32)
    if kind == "uniform":
        V = r.random((n_rows, n_cols))
    else:
        V = r.standard_normal((n_rows, n_cols))
    if kind == "mixed":
        u = r.random((n_rows, n_cols))
        V[u < 0.05] = 0.0
        V[(u >= 0.05) & (u < 0.08)] = -0.0
        V[(u >= 0.08) & (u < 0.09)] *= 1e30
        V[(u >= 0.09) & (u < 0.10)] *= 1e-30
        if n_rows > 2:
            V[r.integers(0, n_rows)] = 0.0
    M[:, :n_cols] = V.astype(np.float32)
    return M, lda


def random_vector(n, seed, kind="normal"):
    r = np.random.default_rng(seed)
    if kind == "uniform":
        v = r.random(n)
    else:
        v = r.standard_normal(n)
    if kind == "mixed":
        u = r.random(n)
        v[u < 0.05] = 0.0
        v[(u >= 0.05) & (u < 0.08)] = -0.0
    return v.astype(np.float32)


def stochastic_pca(N=10**6, D=10, gap=0.1, seed=7):
    """The synthetic eigen-gap dataset of the paper's stochastic-PCA comparison: X = U Sigma V^T with
    random orthonormal U (N x D), V (D x D) and Sigma = diag(1, sqrt(1 - gap), ..., sqrt(1 - gap)), so
    C = X^T X has eigen-gap `gap`.  Returns X (fp32, one cast) and u1 = V[:, 0] (fp64).  Input recipe only."""
    g = np.random.default_rng(seed)
    U, _ = np.linalg.qr(g.standard_normal((N, D)))
    V, _ = np.linalg.qr(g.standard_normal((D, D)))
    sig = np.array([1.0] + [np.sqrt(1.0 - gap)] * (D - 1))
    return ((U * sig) @ V.T).astype(np.float32), V[:, 0].copy()


def batch_draws(N, T, s, seed=8):
    """Algorithm 3 step 3: T mini-batches of s i.i.d. uniform row indices (with replacement), int32."""
    return np.random.default_rng(seed).integers(0, N, (T, s)).astype(np.int32)
