"""Literal-definition brute force (TEST INFRASTRUCTURE) used to pin ``oracle.c``.

Written independently of ``oracle.c``: pure-Python scalar loops over the paper's formulas
exactly as printed, for tiny inputs (n <= 8 for the dense path, n <= 200 for the dense
Google matrix).  Python floats are IEEE fp64.

Citation keys: ``P:n`` = PAPER.md line n; ``S:n`` = SPEC.md line n.
"""
from __future__ import annotations

import math

import numpy as np


def sign(v: float) -> int:
    """sign(.) with sign(0) = 0 (the paper leaves sign(0) undefined)."""
    if v > 0:
        return 1
    if v < 0:
        return -1
    return 0


def min1(w, x) -> float:
    """Eq.(3): sum_i sign(w_i x_i) min(|w_i|, |x_i|) — sign of the product itself."""
    total = 0.0
    for wi, xi in zip(w, x):
        total += sign(float(wi) * float(xi)) * min(abs(float(wi)), abs(float(xi)))
    return total


def min2(w, x) -> float:
    """Eq.(4): sum_i 1(sign(w_i) = sign(x_i)) min(|w_i|, |x_i|)."""
    total = 0.0
    for wi, xi in zip(w, x):
        if sign(float(wi)) == sign(float(xi)):
            total += min(abs(float(wi)), abs(float(xi)))
    return total


def diamond(w, x) -> float:
    """Eq.(9): sum_i (sign(x_i) y_i + x_i sign(y_i)), reading y == w."""
    total = 0.0
    for wi, xi in zip(w, x):
        total += sign(float(xi)) * float(wi) + float(xi) * sign(float(wi))
    return total


def dot(w, x) -> float:
    total = 0.0
    for wi, xi in zip(w, x):
        total += float(wi) * float(xi)
    return total


OPS = {"min1": min1, "min2": min2, "diamond": diamond, "dot": dot}


def matvec(A, x, op="min1"):
    """Matrix extension: entry j = (row j of A) (op) x."""
    f = OPS[op]
    return [f(list(row), list(x)) for row in np.asarray(A, dtype=np.float64)]


def mapi(A, b0, iters, op="min1"):
    """Algorithm 1, literally: w_{t+1} = A (op) w_t ; w_{t+1} /= ||w_{t+1}||_1."""
    w = [float(v) for v in b0]
    norms = []
    for _ in range(iters):
        y = matvec(A, w, op)
        s = 0.0
        for v in y:
            s += abs(v)
        norms.append(s)
        w = [v / s for v in y]
    return w, norms


def rpi(A, b0, iters):
    """Eq.(1): b <- Ab / ||Ab||_2."""
    b = [float(v) for v in b0]
    for _ in range(iters):
        y = matvec(A, b, "dot")
        s = math.sqrt(sum(v * v for v in y))
        b = [v / s for v in y]
    return b


def google_matrix(n, edges, alpha=0.85):
    """Eq.(13), reading Q10: G = alpha H + (1-alpha)/n 1 with H column-stochastic,
    H[i][j] = 1/outdeg(j) for each distinct edge j -> i, dangling columns uniform 1/n."""
    edges = sorted(set((int(s), int(d)) for s, d in edges))
    outdeg = [0] * n
    for s, _ in edges:
        outdeg[s] += 1
    H = np.zeros((n, n))
    for s, d in edges:
        H[d, s] = 1.0 / outdeg[s]
    for j in range(n):
        if outdeg[j] == 0:
            H[:, j] = 1.0 / n
    return alpha * H + (1.0 - alpha) / n * np.ones((n, n))


def rank_dense(n, edges, alpha=0.85, iters=20, b0=None):
    """MAPI ranking by brute force over the materialised G:
    y_i = sum_j sign(G_ij w_j) min(|G_ij|, |w_j|), then Algorithm 1's l1 normalisation."""
    G = google_matrix(n, edges, alpha)
    w = np.full(n, 1.0 / n) if b0 is None else np.asarray(b0, dtype=np.float64).copy()
    deltas = []
    for _ in range(iters):
        y = np.sum(np.sign(G * w[None, :]) * np.minimum(np.abs(G), np.abs(w)[None, :]), axis=1)
        wn = y / np.sum(np.abs(y))
        deltas.append(float(np.sum(np.abs(wn - w))))
        w = wn
    return w, deltas


def google_mavp(n, edges, w, alpha=0.85):
    """One dense G (min1) w product (the literal definition), for w >= 0."""
    G = google_matrix(n, edges, alpha)
    w = np.asarray(w, dtype=np.float64)
    return np.sum(np.sign(G * w[None, :]) * np.minimum(np.abs(G), np.abs(w)[None, :]), axis=1)


def google_dot(n, edges, w, alpha=0.85):
    """One dense G w product (Eq. 1 on the materialised Google matrix)."""
    return google_matrix(n, edges, alpha) @ np.asarray(w, dtype=np.float64)


def pagerank_eig(n, edges, alpha=0.85):
    """The PageRank vector: the eigenvector of the dense G for its eigenvalue 1 (LAPACK geev), l1-unit and
    non-negative (Perron-Frobenius: G is positive and column-stochastic)."""
    G = google_matrix(n, edges, alpha)
    vals, vecs = np.linalg.eig(G)
    k = int(np.argmin(np.abs(vals - 1.0)))
    v = np.real(vecs[:, k])
    return v / v.sum()


def minibatch_mapi(X, batch, beta, w0, gram="min1"):
    """Algorithm 3 written out literally for tiny inputs: per iteration the batch mean of the
    samples' matrices A~_i[j][k] = x_ij (gram) x_ik, w_{t+1} = M (.) w_t - beta w_{t-1} with (.) the min1
    product of Eq. (3), then both w_t and w_{t+1} divided by ||w_{t+1}||_1 (step 5 verbatim).
    Returns (w_T, [||w_{t+1}||_1 for each t])."""
    term = OPS[gram]
    D = len(w0)
    w = [float(v) for v in w0]
    wp = [0.0] * D
    norms = []
    for row_ids in batch:
        s = len(row_ids)
        M = [[0.0] * D for _ in range(D)]
        for i in row_ids:
            x = [float(v) for v in X[i]]
            for j in range(D):
                for k in range(D):
                    M[j][k] += term([x[j]], [x[k]])
        M = [[M[j][k] / s for k in range(D)] for j in range(D)]
        y = [min1(M[j], w) - beta * wp[j] for j in range(D)]
        st = sum(abs(v) for v in y)
        norms.append(st)
        wp = [v / st for v in w]
        w = [v / st for v in y]
    return np.array(w), np.array(norms)
