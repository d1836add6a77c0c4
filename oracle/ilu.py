"""NEXT-2 — the paper's smoother: ILU(0) (PAPER.md:243 "apply a smoother", :408 "ILU(0)";
SPEC.md:59-76), in red-black cell ordering (reading B12).

ILU(0) (Saad, Iterative Methods, Alg. 10.4, IKJ variant) of the matrix P A P^T, where P
orders the "red" cells (i + j + k even) first and the "black" cells after them, each
group in natural order: L unit lower and U upper with the sparsity of A's lower and
upper parts, (L U)_ij = A_ij on A's pattern.  One smoothing step is
x <- x + (L U)^{-1} (b - A x) (undamped, ν steps).

Written the plain way: a row-by-row IKJ elimination restricted to the pattern (pure
Python loops: small grids only), and scipy's triangular solves.
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular


def rb_permutation(nx, ny, nz):
    """perm[new] = old: red cells (i + j + k even) first, then black, natural order."""
    c = np.arange(nx * ny * nz)
    i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
    red = (i + j + k) % 2 == 0
    return np.concatenate([c[red], c[~red]])


def ilu0(A):
    """IKJ ILU(0) of a square CSR matrix in its given ordering: returns (L, U) with L unit
    lower triangular (diagonal stored) and U upper triangular, both on A's pattern."""
    A = sp.csr_matrix(A)
    A.sort_indices()
    n = A.shape[0]
    rows = [dict(zip(A.indices[A.indptr[i]:A.indptr[i + 1]].tolist(),
                     A.data[A.indptr[i]:A.indptr[i + 1]].tolist())) for i in range(n)]
    for i in range(n):
        ri = rows[i]
        for k in sorted(c for c in ri if c < i):
            if rows[k].get(k, 0.0) == 0.0:
                raise ZeroDivisionError("zero pivot in ILU(0)")
            ri[k] = ri[k] / rows[k][k]
            lik = ri[k]
            for j, ukj in rows[k].items():
                if j > k and j in ri:
                    ri[j] = ri[j] - lik * ukj
    Lr, Lc, Lv, Ur, Uc, Uv = [], [], [], [], [], []
    for i, ri in enumerate(rows):
        for j, v in ri.items():
            if j < i:
                Lr.append(i), Lc.append(j), Lv.append(v)
            else:
                Ur.append(i), Uc.append(j), Uv.append(v)
        Lr.append(i), Lc.append(i), Lv.append(1.0)
    L = sp.csr_matrix((Lv, (Lr, Lc)), shape=(n, n))
    U = sp.csr_matrix((Uv, (Ur, Uc)), shape=(n, n))
    return L, U


class RBILU0:
    """(L U)^{-1} of the red-black ordered ILU(0) of A."""

    def __init__(self, A, nx, ny, nz):
        self.perm = rb_permutation(nx, ny, nz)
        Ap = sp.csr_matrix(A)[self.perm][:, self.perm]
        self.L, self.U = ilu0(Ap)

    def solve(self, r):
        rp = np.asarray(r, dtype=np.float64)[self.perm]
        y = spsolve_triangular(self.L, rp, lower=True)
        e = spsolve_triangular(self.U, y, lower=False)
        out = np.empty_like(e)
        out[self.perm] = e
        return out


def smooth(A, b, x, fact, nu):
    """ν undamped ILU(0) smoothing steps x <- x + (LU)^{-1}(b - A x)."""
    for _ in range(nu):
        x = x + fact.solve(b - A @ x)
    return x
