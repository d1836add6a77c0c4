"""NEXT-1 — flexible GMRES with the multibasis cycle as preconditioner (oracle).

PAPER.md:287 ("the multiscale solver can be used ... as a preconditioner for GMRES"),
SPEC.md:95-103 (restarted GMRES with right preconditioning).  The
preconditioner M^{-1} v is ONE iteration of Eq. (8) (oracle.cycle.stage over the static
levels) applied to the right-hand side v from a zero initial guess; "flexible"
(Saad's FGMRES) because z_j = M^{-1} v_j is stored explicitly, so a preconditioner that
changes between steps stays admissible.

Algorithm (restart m, textbook order):
    r0 = b - A x0, beta = ||r0||, v_1 = r0 / beta, g = beta e_1
    for j = 1..m:
        z_j = M^{-1} v_j ;  w = A z_j
        for i = 1..j:  h_ij = (w, v_i) ;  w = w - h_ij v_i          (modified Gram-Schmidt)
        h_{j+1,j} = ||w|| ;  v_{j+1} = w / h_{j+1,j}
        apply the previous Givens rotations to column j of H, build rotation j,
        g_{j+1} = -s_j g_j, g_j = c_j g_j;  |g_{j+1}| = ||b - A x_j||
        stop the cycle when |g_{j+1}| <= tol ||b||
    y = H(1:j,1:j)^{-1} g(1:j) (back substitution) ;  x = x0 + Z y ;  restart with x0 = x
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .cycle import stage


def precondition(A, DA, v, levels, omega_s=2.0 / 3.0, nu=1, post=False, smoother=None):
    """z = M^{-1} v: one multibasis cycle (Eq. 8) from x = 0 with right-hand side v."""
    z = np.zeros_like(v)
    for lev in levels:
        z = stage(A, DA, v, z, lev, omega_s, nu, post, smoother)
    return z


def fgmres(A, b, x0, levels, omega_s=2.0 / 3.0, nu=1, post=False, tol=1e-6, restart=30,
           max_iter=1000, fixed_iters=0, precond=None, smoother=None):
    """Returns dict(x, iters, res (true relative residual at each restart start and the
    Arnoldi estimate after each step), converged).  precond: optional callable v -> z
    replacing the multibasis cycle (pins: identity, exact inverse)."""
    A = sp.csr_matrix(A)
    DA = A.diagonal()
    x = np.array(x0, dtype=np.float64, copy=True)
    bnorm = float(np.linalg.norm(b))
    scale = bnorm if bnorm > 0 else 1.0
    res = []
    k = 0
    converged = False
    target = fixed_iters if fixed_iters > 0 else max_iter
    while True:
        r = b - A @ x
        beta = float(np.linalg.norm(r))
        if k == 0:
            res.append(beta / scale)
        if fixed_iters <= 0 and beta / scale <= tol:
            converged = True
            break
        if k >= target or beta == 0.0:
            break
        m = restart
        V = np.zeros((len(b), m + 1))
        Z = np.zeros((len(b), m))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[:, 0] = r / beta
        j_used = 0
        for j in range(m):
            Z[:, j] = (precond(V[:, j]) if precond is not None
                       else precondition(A, DA, V[:, j], levels, omega_s, nu, post, smoother))
            w = A @ Z[:, j]
            for i in range(j + 1):
                H[i, j] = float(w @ V[:, i])
                w = w - H[i, j] * V[:, i]
            H[j + 1, j] = float(np.linalg.norm(w))
            if H[j + 1, j] != 0.0:
                V[:, j + 1] = w / H[j + 1, j]
            for i in range(j):  # previous rotations on column j
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            d = np.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / d if d != 0.0 else 1.0
            sn[j] = H[j + 1, j] / d if d != 0.0 else 0.0
            H[j, j] = d
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            k += 1
            j_used = j + 1
            res.append(abs(g[j + 1]) / scale)
            if fixed_iters > 0:
                if k >= fixed_iters:
                    break
            elif abs(g[j + 1]) / scale <= tol or k >= max_iter:
                break
        y = np.zeros(j_used)
        for i in range(j_used - 1, -1, -1):  # back substitution
            y[i] = (g[i] - H[i, i + 1:j_used] @ y[i + 1:j_used]) / H[i, i]
        x = x + Z[:, :j_used] @ y
        if fixed_iters > 0 and k >= fixed_iters:
            break
    out = dict(x=x, iters=k, res=np.array(res))
    final = float(np.linalg.norm(b - A @ x)) / scale
    out["true_res"] = final
    out["converged"] = converged or final <= tol
    return out
