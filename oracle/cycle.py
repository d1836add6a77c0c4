"""O9–O11 — the iterative multiscale multibasis solver (Richardson).

Eq. (8), for ℓ = 1..N_p in order:
    x <- x + S^ℓ(A, q - A x)                              (smoothing)
    x <- x + P^ℓ (A_c^ℓ)^{-1} R^ℓ (q - A x),  R^ℓ = P^ℓT     (coarse correction, :241, :225)
with S^ℓ = ν sweeps of damped Jacobi x <- x + ω_s D_A^{-1}(b - A x) (reading A9;
the paper's own smoother is ILU(0)).  `post=True` swaps the two
steps inside each stage (reading A10, BASELINE.json configs[2]).

Stop test (O10): after each full cycle k, ρ_k = ||b - A x||_2/||b||_2;
stop when ρ_k <= tol (count = k) or k = max_iter; `fixed_iters > 0` runs exactly
that many cycles.  Divergence when ||r_k|| > 1e6 ||r_0||.

Dynamic stage (O11; readings A12, A14, A15): for
k >= 2, Δp = x_start(k) - x_start(k-1), the Δp-binned constant-basis partition
of oracle.partition.dynamic_partition becomes an extra stage appended after the
static stages of iteration k (skipped when max|Δp| = 0).
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .coarse import CoarseSolver, galerkin
from .partition import dynamic_partition


class Level:
    """One (P, R = P^T, A_c) stage.  coarse / assoc select an alternate exact coarse
    solver / summation order (oracle.coarse; floor measurement only)."""

    def __init__(self, P, A, coarse="lu", assoc="right"):
        self.P = sp.csr_matrix(P)
        self.PT = self.P.T.tocsr()
        self.Ac = galerkin(self.P, A, assoc)
        self.solver = CoarseSolver(self.Ac, coarse)

    @property
    def M(self):
        return self.P.shape[1]


def constant_basis(part, M):
    """P_ij = 1 iff part[i] = j (PAPER.md:260 caption)."""
    N = len(part)
    return sp.csr_matrix((np.ones(N), (np.arange(N), part)), shape=(N, M))


def residual(A, b, x):
    return b - A @ x


def jacobi(A, DA, b, x, omega_s, nu):
    for _ in range(nu):
        x = x + omega_s * (residual(A, b, x) / DA)
    return x


def coarse_correction(A, b, x, level):
    r = residual(A, b, x)
    rc = level.PT @ r
    xc = level.solver.solve(rc)
    return x + level.P @ xc


def smooth_step(A, DA, b, x, omega_s, nu, smoother=None):
    """The stage smoother: damped Jacobi (reading A9) or, given an ILU(0) factor object
    (oracle.ilu.RBILU0, NEXT-2), ν undamped ILU(0) steps."""
    if smoother is None:
        return jacobi(A, DA, b, x, omega_s, nu)
    for _ in range(nu):
        x = x + smoother.solve(residual(A, b, x))
    return x


def stage(A, DA, b, x, level, omega_s, nu, post, smoother=None):
    if post:
        x = coarse_correction(A, b, x, level)
        return smooth_step(A, DA, b, x, omega_s, nu, smoother)
    x = smooth_step(A, DA, b, x, omega_s, nu, smoother)
    return coarse_correction(A, b, x, level)


def iterate(A, b, x0, levels, omega_s=2.0 / 3.0, nu=1, post=False, tol=1e-6,
            max_iter=1000, fixed_iters=0, dynamic=None, record_dynamic=False, smoother=None,
            coarse="lu", assoc="right"):
    """Run the multibasis Richardson iteration.

    dynamic: None or dict(nx=, ny=, nz=, edges=(0.1, 0.5), max_blocks=1024).
    record_dynamic: True keeps every (k, part, M) in out["dyn"]; a callable is called
    with (k, part, M) instead.
    coarse / assoc: alternate coarse solver / A_c summation order for the dynamic
    stage's levels (oracle.coarse; floor measurement only).
    Returns dict(x, iters, res (ρ_0..ρ_k), converged, diverged, dyn=[(k, part, M)])."""
    A = sp.csr_matrix(A)
    DA = A.diagonal()
    x = np.array(x0, dtype=np.float64, copy=True)
    bnorm = float(np.linalg.norm(b))
    scale = bnorm if bnorm > 0 else 1.0
    r0 = float(np.linalg.norm(residual(A, b, x)))
    res = [r0 / scale]
    out = dict(converged=False, diverged=False, dyn=[], dyn_M=[])
    k = 0
    if fixed_iters <= 0 and res[0] <= tol:
        out.update(x=x, iters=0, res=np.array(res), converged=True)
        return out
    n_target = fixed_iters if fixed_iters > 0 else max_iter
    x_prev_start = None
    while k < n_target:
        k += 1
        x_start = x.copy()
        stages = list(levels)
        if dynamic is not None and k >= 2:
            dp = x_start - x_prev_start
            part, M = dynamic_partition(dp, dynamic["nx"], dynamic["ny"], dynamic["nz"],
                                        dynamic.get("edges", (0.1, 0.5)),
                                        dynamic.get("max_blocks", 1024))
            out["dyn_M"].append(M)
            if part is not None:
                stages.append(Level(constant_basis(part, M), A, coarse, assoc))
                if callable(record_dynamic):
                    record_dynamic(k, part, M)
                elif record_dynamic:
                    out["dyn"].append((k, part, M))
        x_prev_start = x_start
        for lev in stages:
            x = stage(A, DA, b, x, lev, omega_s, nu, post, smoother)
        rk = float(np.linalg.norm(residual(A, b, x)))
        res.append(rk / scale)
        if rk > 1e6 * r0 and r0 > 0:
            out["diverged"] = True
            break
        if fixed_iters <= 0 and res[-1] <= tol:
            out["converged"] = True
            break
    out.update(x=x, iters=k, res=np.array(res))
    if fixed_iters > 0:
        out["converged"] = res[-1] <= tol
    return out
