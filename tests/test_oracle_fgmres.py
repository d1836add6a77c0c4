"""Oracle pins — flexible GMRES (NEXT-1).

With the identity preconditioner FGMRES is GMRES, whose k-th iterate is the unique
minimiser of ||b - A x|| over x0 + K_k(A, r0): checked against a brute-force Krylov
least-squares solve (numpy QR + lstsq).  Its Arnoldi residual estimates |g_{j+1}| equal
the true residual norms.  The exact preconditioner A^{-1} converges in one step; an n x n
system converges in <= n steps; with the multibasis cycle it converges far faster than
Richardson, to the direct solve.
"""
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import fgmres as og
from oracle import pipeline, tpfa
from oracle.cycle import Level
from synth.configs import make_problem, random_problem


def _small_spd(n=40, seed=0):
    rng = np.random.default_rng(seed)
    B = sp.random(n, n, density=0.15, random_state=seed)
    A = (B @ B.T + sp.diags(rng.uniform(1.0, 3.0, n))).tocsr()
    return A, rng.standard_normal(n)


def _krylov_min_residual(A, b, x0, k):
    r0 = b - A @ x0
    K = np.zeros((len(b), k))
    v = r0.copy()
    for j in range(k):
        K[:, j] = v
        v = A @ v
    Q, _ = np.linalg.qr(K)
    y, *_ = np.linalg.lstsq(A @ Q, r0, rcond=None)
    return x0 + Q @ y


def test_identity_preconditioner_is_gmres_minimiser():
    A, b = _small_spd()
    x0 = np.zeros_like(b)
    for k in (1, 3, 7):
        out = og.fgmres(A, b, x0, [], tol=0.0, restart=50, fixed_iters=k, precond=lambda v: v)
        ref = _krylov_min_residual(A, b, x0, k)
        assert np.linalg.norm(out["x"] - ref) <= 1e-9 * np.linalg.norm(ref), k


def test_arnoldi_estimate_equals_true_residual():
    A, b = _small_spd(30, 1)
    x0 = np.zeros_like(b)
    for k in (2, 5, 9):
        out = og.fgmres(A, b, x0, [], tol=0.0, restart=50, fixed_iters=k, precond=lambda v: v)
        true = np.linalg.norm(b - A @ out["x"]) / np.linalg.norm(b)
        assert abs(out["res"][-1] - true) <= 1e-12 + 1e-9 * true


def test_exact_preconditioner_one_step():
    A, b = _small_spd(25, 2)
    lu = spla.splu(A.tocsc())
    out = og.fgmres(A, b, np.zeros_like(b), [], tol=1e-12, restart=10, precond=lu.solve)
    assert out["iters"] == 1 and out["converged"]


def test_n_steps_for_n_unknowns():
    A, b = _small_spd(12, 3)
    out = og.fgmres(A, b, np.zeros_like(b), [], tol=1e-11, restart=12, precond=lambda v: v)
    assert out["converged"] and out["iters"] <= 12


def test_multibasis_preconditioner_beats_richardson():
    prob = make_problem(1, max_sweeps=60)
    orc = pipeline.run(prob, max_iter=5000)
    A, q = orc["A"], orc["q"]
    out = og.fgmres(A, q, np.zeros(prob.N), orc["levels"], prob.omega_s, prob.nu,
                    prob.post_smooth, tol=1e-6, restart=30, max_iter=2000)
    assert out["converged"]
    assert out["iters"] < orc["sol"]["iters"] / 3, (out["iters"], orc["sol"]["iters"])
    p = spla.spsolve(A.tocsc(), q)
    assert np.linalg.norm(out["x"] - p) <= 1e-4 * np.linalg.norm(p)


def test_restart_and_fixed_iterations():
    prob = random_problem(3, 14, 11, 4, (4, 4, 2), sigma=1.0, max_sweeps=20)
    orc = pipeline.run(prob, max_iter=3000)
    A, q = orc["A"], orc["q"]
    full = og.fgmres(A, q, np.zeros(prob.N), orc["levels"], tol=1e-10, restart=8, max_iter=400)
    assert full["converged"]
    fix = og.fgmres(A, q, np.zeros(prob.N), orc["levels"], tol=1e-10, restart=8, fixed_iters=5)
    assert fix["iters"] == 5 and len(fix["res"]) == 6
