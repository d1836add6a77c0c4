"""O8 — Galerkin coarse operator and its direct solve.

PAPER.md:212-216 (Eq. pressure_system_reduced: A_c = R A P, q_c = R q);
PAPER.md:225 (Galerkin restriction R = P^T); PAPER.md:410 ("inverting the coarse
matrix ... O(M^p) ... worst case p = 3 for a dense matrix inverted by direct
Gaussian elimination"); SPEC.md:77-85 (dense LU with partial pivoting, singular
if a pivot is below 1e-14 * max|A|).

The oracle's solver is dense `scipy.linalg.lu_factor` when M <= DENSE_MAX, else
sparse `splu` (method "lu").  The other methods are ALTERNATE exact direct solvers
of the same SPD system, used only to measure the rounding floor of the method
(DESIGN.md §3.5): the Richardson iteration amplifies O(eps) differences of the
coarse solve by cond(A_c), so the distance between two backward-stable solvers is
the yardstick any third implementation (the GPU's) is held to.  Each is one
library call, no arithmetic of its own:
    "cholesky"      LAPACK potrf/potrs (dense) or banded Cholesky pbtrf/pbtrs on the
                    natural-order band (sparse M; the band solver of SURVEY §8.a5)
    "inverse"       LAPACK getrf/getri explicit inverse + GEMV (reading B1; the sparse A_c
                    densified first)
    "lu_reversed"   LU of the coarse matrix with its unknowns in reverse order (LAPACK
                    dense; SuperLU, natural order, sparse)
    "splu_natural"  SuperLU with natural column order
Every method works for dense (M <= DENSE_MAX) and sparse A_c.
`galerkin(..., assoc="left")` forms (P^T A) P instead of P^T (A P): another
summation order of the same product.
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as la
import scipy.sparse as sp
import scipy.sparse.linalg as spla

DENSE_MAX = 4096
METHODS = ("lu", "cholesky", "inverse", "lu_reversed", "splu_natural")


class SingularCoarse(Exception):
    pass


def galerkin(P, A, assoc="right"):
    """A_c = P^T A P (scipy sparse products); dense ndarray when M <= DENSE_MAX.
    assoc="right": P^T (A P) (the oracle); "left": (P^T A) P (alternate order)."""
    P = sp.csr_matrix(P)
    if assoc == "right":
        Ac = (P.T @ (A @ P)).tocsr()
    elif assoc == "left":
        Ac = ((P.T.tocsr() @ A) @ P).tocsr()
    else:
        raise ValueError(assoc)
    if Ac.shape[0] <= DENSE_MAX:
        return Ac.toarray()
    Ac.sort_indices()
    return Ac


def _banded_lower(Ac):
    """Lower band storage ab[k, j] = A[j + k, j] (LAPACK 'L' layout) of a sparse SPD."""
    coo = sp.tril(Ac).tocoo()
    bw = int(np.max(coo.row - coo.col)) if coo.nnz else 0
    ab = np.zeros((bw + 1, Ac.shape[0]))
    ab[coo.row - coo.col, coo.col] = coo.data
    return ab


class CoarseSolver:
    def __init__(self, Ac, method="lu"):
        if method not in METHODS:
            raise ValueError(method)
        self.Ac = Ac
        self.M = Ac.shape[0]
        self.method = method
        self._dense = isinstance(Ac, np.ndarray)
        if self._dense:
            amax = np.max(np.abs(Ac)) if Ac.size else 0.0
            lu, piv = la.lu_factor(Ac, check_finite=True)
            if self.M == 0 or np.min(np.abs(np.diag(lu))) < 1e-14 * amax or amax == 0.0:
                raise SingularCoarse("singular coarse matrix (SPEC.md:81)")
            if method == "lu":
                self._f = (lu, piv)
            elif method == "cholesky":
                self._f = la.cho_factor(Ac, lower=True)
            elif method == "inverse":
                self._f = np.linalg.inv(Ac)
            elif method == "lu_reversed":
                self._f = la.lu_factor(Ac[::-1, ::-1])
            else:  # splu_natural
                self._f = spla.splu(sp.csc_matrix(Ac), permc_spec="NATURAL")
        else:
            try:
                if method == "lu":
                    self._f = spla.splu(sp.csc_matrix(Ac))
                elif method == "splu_natural":
                    self._f = spla.splu(sp.csc_matrix(Ac), permc_spec="NATURAL")
                elif method == "cholesky":
                    self._f = la.cholesky_banded(_banded_lower(Ac), lower=True)
                elif method == "inverse":
                    self._f = np.linalg.inv(Ac.toarray())
                else:  # lu_reversed: SuperLU of the coarse matrix with its unknowns reversed
                    self._f = spla.splu(sp.csc_matrix(Ac[::-1][:, ::-1]), permc_spec="NATURAL")
            except RuntimeError as e:  # exactly singular
                raise SingularCoarse(str(e))
            except la.LinAlgError as e:
                raise SingularCoarse(str(e))

    def solve(self, rc):
        m = self.method
        if self._dense:
            if m == "lu":
                return la.lu_solve(self._f, rc)
            if m == "cholesky":
                return la.cho_solve(self._f, rc)
            if m == "inverse":
                return self._f @ rc
            if m == "splu_natural":
                return self._f.solve(rc)
            return la.lu_solve(self._f, rc[::-1])[::-1]
        if m == "cholesky":
            return la.cho_solve_banded((self._f, True), rc)
        if m == "inverse":
            return self._f @ rc
        if m == "lu_reversed":
            return self._f.solve(rc[::-1])[::-1]
        return self._f.solve(rc)
