"""O8 — Galerkin coarse operator and its direct solve.

PAPER.md:212-216 (Eq. pressure_system_reduced: A_c = R A P, q_c = R q);
PAPER.md:225 (Galerkin restriction R = P^T); PAPER.md:410 ("inverting the coarse
matrix ... O(M^p) ... worst case p = 3 for a dense matrix inverted by direct
Gaussian elimination"); SPEC.md:77-85 (dense LU with partial pivoting, singular
if a pivot is below 1e-14 * max|A|).

Dense `scipy.linalg.lu_factor` when M <= DENSE_MAX, else sparse `splu`.
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as la
import scipy.sparse as sp
import scipy.sparse.linalg as spla

DENSE_MAX = 4096


class SingularCoarse(Exception):
    pass


def galerkin(P, A):
    """A_c = P^T A P (scipy sparse products); dense ndarray when M <= DENSE_MAX."""
    P = sp.csr_matrix(P)
    Ac = (P.T @ (A @ P)).tocsr()
    if Ac.shape[0] <= DENSE_MAX:
        return Ac.toarray()
    Ac.sort_indices()
    return Ac


class CoarseSolver:
    def __init__(self, Ac):
        self.Ac = Ac
        self.M = Ac.shape[0]
        if isinstance(Ac, np.ndarray):
            amax = np.max(np.abs(Ac)) if Ac.size else 0.0
            lu, piv = la.lu_factor(Ac, check_finite=True)
            if self.M == 0 or np.min(np.abs(np.diag(lu))) < 1e-14 * amax or amax == 0.0:
                raise SingularCoarse("singular coarse matrix (SPEC.md:81)")
            self._lu = (lu, piv)
            self._sparse = None
        else:
            try:
                self._sparse = spla.splu(sp.csc_matrix(Ac))
            except RuntimeError as e:  # exactly singular
                raise SingularCoarse(str(e))
            self._lu = None

    def solve(self, rc):
        if self._lu is not None:
            return la.lu_solve(self._lu, rc)
        return self._sparse.solve(rc)
