"""O6–O7 — MsRSB restricted-smoothing basis.

The paper cites MsRSB without stating it; the
algorithm follows BASELINE.json north_star ("repeated damped-Jacobi sweeps
P <- P - w D^-1 (A P) on the fixed sparsity pattern of the prolongation,
restricted to each basis function's support region and renormalised to a
partition of unity") and SPEC.md:428-436.  Readings:

A2  the smoothing matrix is the flux matrix A_T (zero row sums, no gauge); D = diag(A_T).
A5  positive form: P̂_ij = (1-ω) P_ij + (ω/D_i) Σ_{l≠i} T_il P_lj  — identical in
    exact arithmetic to P - ω D^-1 A_T P because A_T has zero row sums.
A6  renormalise EVERY row after every sweep: P_ij <- P̂_ij / Σ_k P̂_ik
    (requirement 3).
A16 δ_n = max |P^{n+1} - P^n| after renormalisation; stop when δ_n <= tol or
    n = max_sweeps.

The sweep is written the plain way: Q = Off @ P (scipy SpGEMM, Off = the
nonnegative off-diagonal part of -A_T), then Q is sampled on the pattern.
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


class Basis:
    """P stored as values aligned with a fixed CSR pattern (N x M)."""

    def __init__(self, pattern, vals):
        self.pattern = pattern
        self.rows = np.repeat(np.arange(pattern.shape[0]), np.diff(pattern.indptr))
        self.cols = pattern.indices.astype(np.int64)
        self.vals = vals

    @property
    def shape(self):
        return self.pattern.shape

    def matrix(self):
        return sp.csr_matrix((self.vals, self.pattern.indices, self.pattern.indptr),
                             shape=self.pattern.shape)

    def dense(self):
        return self.matrix().toarray()

    def copy(self):
        return Basis(self.pattern, self.vals.copy())


def indicator(part, pattern):
    """O6: P^0 = indicator of the partition restricted to the pattern."""
    b = Basis(pattern, None)
    b.vals = (b.cols == part[b.rows]).astype(np.float64)
    return b


def sweep(basis, A_T, omega):
    """One restricted-smoothing sweep; returns (new basis, δ)."""
    D = A_T.diagonal()
    if np.any(D == 0.0):
        raise ValueError("zero diagonal in A_T (SPEC.md:432)")
    Off = -(A_T - sp.diags(D)).tocsr()
    Off.eliminate_zeros()
    Q = (Off @ basis.matrix()).tocsr()
    q = np.asarray(Q[basis.rows, basis.cols]).ravel()
    p = basis.vals
    phat = (1.0 - omega) * p + (omega / D[basis.rows]) * q
    rowsum = np.bincount(basis.rows, weights=phat, minlength=basis.shape[0])
    pnew = phat / rowsum[basis.rows]
    delta = float(np.max(np.abs(pnew - p))) if len(p) else 0.0
    return Basis(basis.pattern, pnew), delta


def smooth(basis, A_T, omega=2.0 / 3.0, max_sweeps=300, tol=1e-3, fixed=False):
    """Repeat `sweep` until δ <= tol (unless fixed) or max_sweeps.

    Returns (basis, sweeps_done, deltas)."""
    deltas = []
    b = basis
    for n in range(1, max_sweeps + 1):
        b, d = sweep(b, A_T, omega)
        deltas.append(d)
        if not fixed and d <= tol:
            break
    return b, len(deltas), np.array(deltas)
