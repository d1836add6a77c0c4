"""O2–O3 — two-point flux approximation and the pressure matrix.

PAPER.md:101 ("we use a two-point approximation for the flux terms and
single-point upstream evaluation for the interface mobilities")
(t_i = A_face*K_i/(Δ/2), T_ij = (1/t_i + 1/t_j)^{-1}); PAPER.md:207-211 (A p = q).
Readings: A2 — the basis smooths with the flux matrix A_T (zero
row sums, no gauge); A7 — the solve matrix is A = A_T with A_00 doubled
(pure-Neumann gauge); A8 — A is the positive semidefinite flux matrix, q > 0 is
injection.  TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .grid import all_faces


def half_transmissibility(K, area, dist):
    """t = K * A_face / (Δ/2)."""
    return K * area / (dist / 2.0)


def face_transmissibility(t_left, t_right, mult=1.0, mob=1.0):
    """T_f = (1/t_i + 1/t_l)^{-1} * m_f * λ_f."""
    return 1.0 / (1.0 / t_left + 1.0 / t_right) * mult * mob


def transmissibilities(prob, mob=None):
    """Per-axis lists of (left, right, T) for every interior face.

    `mob` is an optional list of three per-face mobility arrays (config 4)."""
    if np.any(prob.kx <= 0) or np.any(prob.ky <= 0) or np.any(prob.kz <= 0):
        raise ValueError("nonpositive permeability (SPEC.md:163)")
    faces = all_faces(prob.nx, prob.ny, prob.nz)
    K = (prob.kx, prob.ky, prob.kz)
    d = (prob.dx, prob.dy, prob.dz)
    area = (prob.dy * prob.dz, prob.dx * prob.dz, prob.dx * prob.dy)
    mults = (prob.mult_x, prob.mult_y, prob.mult_z)
    out = []
    for a in range(3):
        left, right = faces[a]
        tl = half_transmissibility(K[a][left], area[a], d[a])
        tr = half_transmissibility(K[a][right], area[a], d[a])
        m = mults[a] if mults[a] is not None else np.ones(len(left))
        lam = mob[a] if mob is not None else np.ones(len(left))
        out.append((left, right, face_transmissibility(tl, tr, m, lam)))
    return out


def flux_matrix(N, trans, diag_order="assembly"):
    """A_T = Σ_f T_f (e_i - e_l)(e_i - e_l)^T, a scipy CSR matrix.

    diag_order="faces" is an ALTERNATE summation order of the same diagonal (floor
    measurement only): D_i summed over the cell's faces left to right in
    ascending neighbour index, instead of scipy's duplicate-summing order.  The sums agree
    to an ulp or two, but ILU(0)'s black pivots cancel against them (reading B12)."""
    rows, cols, vals = [], [], []
    for left, right, T in trans:
        rows += [left, right, left, right]
        cols += [left, right, right, left]
        vals += [T, T, -T, -T]
    if rows:
        rows = np.concatenate(rows)
        cols = np.concatenate(cols)
        vals = np.concatenate(vals)
    else:
        rows = cols = np.zeros(0, dtype=np.int64)
        vals = np.zeros(0)
    A = sp.coo_matrix((vals, (rows, cols)), shape=(N, N)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    if diag_order == "faces":
        cell = np.concatenate([t[0] for t in trans] + [t[1] for t in trans]) if trans else []
        nbr = np.concatenate([t[1] for t in trans] + [t[0] for t in trans]) if trans else []
        tv = np.concatenate([t[2] for t in trans] * 2) if trans else []
        order = np.lexsort((nbr, cell))
        D = np.zeros(N)
        np.add.at(D, np.asarray(cell)[order], np.asarray(tv)[order])  # sequential, in order
        A.setdiag(D)
    elif diag_order != "assembly":
        raise ValueError(diag_order)
    return A


def gauge(A_T):
    """Solve matrix A: A_T with A_00 doubled (reading A7).  For Σq = 0 the unique
    solution of A p = q is the Neumann solution with p_0 = 0."""
    A = A_T.tocsr(copy=True)
    A.sort_indices()
    row0 = slice(A.indptr[0], A.indptr[1])
    pos = np.nonzero(A.indices[row0] == 0)[0]
    if len(pos):
        A.data[A.indptr[0] + pos[0]] = 2.0 * A.data[A.indptr[0] + pos[0]]
    return A


def build(prob, mob=None, diag_order="assembly"):
    """Return (A_T, A, q, trans) for a synth.Problem (diag_order: flux_matrix)."""
    trans = transmissibilities(prob, mob)
    A_T = flux_matrix(prob.N, trans, diag_order)
    A = gauge(A_T)
    q = prob.rhs()
    return A_T, A, q, trans
