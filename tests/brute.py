"""Brute-force / library references used to PIN the oracle (tests only).

Each routine here is either a textbook brute force on tiny inputs or a call
into an independent library routine (scipy.sparse.csgraph, numpy.linalg), and
builds its matrices from the input TUPLES, not from the CSR the oracle reads —
so a CSR indexing slip (in vs out, transposed operand) in the oracle shows up.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse import csgraph

INF = 0xFFFFFFFF


def tuples_of(g):
    """Directed edge list (src, dst, w) of a simgen CSR (rows [0,n))."""
    deg = np.diff(g.row_ptr).astype(np.int64)
    src = np.repeat(np.arange(g.n, dtype=np.int64), deg)
    dst = g.col.astype(np.int64)
    w = np.ones_like(dst) if g.w is None else g.w.astype(np.int64)
    return src, dst, w


def min_weight_matrix(n, src, dst, w):
    """Dense matrix of min weight per (u,v) with duplicates collapsed by min (scipy would sum)."""
    W = np.full((n, n), np.inf)
    for a, b, c in zip(src, dst, w):
        if c < W[a, b]:
            W[a, b] = c
    return W


def bfs_levels_scipy(n, src, dst, s):
    A = sp.csr_matrix((np.ones(len(src)), (src, dst)), shape=(n, n))
    d = csgraph.shortest_path(A, directed=True, unweighted=True, indices=[s])[0]
    return np.where(np.isinf(d), INF, d).astype(np.uint32)


def floyd_warshall(n, src, dst, w, s):
    W = min_weight_matrix(n, src, dst, w)
    D = W.copy()
    np.fill_diagonal(D, 0)
    for k in range(n):
        D = np.minimum(D, D[:, k:k + 1] + D[k:k + 1, :])
    d = D[s]
    return np.where(np.isinf(d), INF, d).astype(np.uint32)


def dijkstra_scipy(n, src, dst, w, s):
    W = min_weight_matrix(n, src, dst, w)
    rr, cc = np.nonzero(np.isfinite(W))
    A = sp.csr_matrix((W[rr, cc], (rr, cc)), shape=(n, n))
    d = csgraph.dijkstra(A, directed=True, indices=[s])[0]
    return np.where(np.isinf(d), INF, d).astype(np.uint32)


def peel(n, src, dst, k):
    """Exhaustive peeling: delete vertices of (multigraph) degree < k until stable."""
    alive = np.ones(n, bool)
    while True:
        m = alive[src] & alive[dst]
        deg = np.bincount(src[m], minlength=n)
        kill = alive & (deg < k)
        if not kill.any():
            return alive
        alive &= ~kill


def coreness_by_peeling(n, src, dst):
    core = np.zeros(n, np.int64)
    k = 1
    while True:
        alive = peel(n, src, dst, k)
        if not alive.any():
            return core.astype(np.uint32)
        core[alive] = k
        k += 1


def pagerank_eigvec(n, src, dst, d):
    """Stationary vector of the Google matrix with dangling redistribution (numpy.linalg.eig)."""
    outdeg = np.bincount(src, minlength=n).astype(float)
    P = np.zeros((n, n))
    for a, b in zip(src, dst):
        P[b, a] += 1.0 / outdeg[a]
    P[:, outdeg == 0] = 1.0 / n
    G = d * P + (1 - d) / n * np.ones((n, n))
    vals, vecs = np.linalg.eig(G)
    i = int(np.argmin(np.abs(vals - 1.0)))
    v = np.real(vecs[:, i])
    return v / v.sum()


def pagerank_linear_solve(n, src, dst, d, variant):
    """Exact fixed point of the PageRank recurrence by a dense linear solve
    (numpy.linalg.solve), matrices from the tuples.
    variant 0: r = (1-d)/n + d (P r + (e_dang . r)/n)   (column-stochastic, dangling redistributed)
    variant 1: r = (1-d) + d P r                          (dangling dropped)"""
    outdeg = np.bincount(src, minlength=n).astype(float)
    P = np.zeros((n, n))
    for a, b in zip(src, dst):
        P[b, a] += 1.0 / outdeg[a]
    if variant == 0:
        P[:, outdeg == 0] = 1.0 / n
        return np.linalg.solve(np.eye(n) - d * P, np.full(n, (1 - d) / n))
    return np.linalg.solve(np.eye(n) - d * P, np.full(n, 1 - d))


def spmv_dense(n, src, dst, w, x):
    A = np.zeros((n, n))
    for a, b, c in zip(src, dst, w):
        A[a, b] += c
    return A.T.astype(np.float64) @ x.astype(np.float64)
