"""Pins for the NEXT-2 oracle smoother (oracle/ilu.py): ILU(0) by its defining property
((LU)_ij = A_ij on A's pattern, L unit lower / U upper on A's pattern), exactness where
ILU(0) has no fill, the red-black closed form of the factors, and contraction."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import ilu
from oracle import pipeline as opl
from oracle import tpfa
from synth.configs import make_problem, random_problem


def _tridiag(n, seed=0):
    rng = np.random.default_rng(seed)
    off = -rng.uniform(0.5, 2.0, n - 1)
    d = np.zeros(n)
    d[:-1] -= off
    d[1:] -= off
    d += rng.uniform(0.1, 1.0, n)
    return sp.diags([off, d, off], [-1, 0, 1], format="csr")


def test_ilu0_exact_without_fill():
    """A tridiagonal matrix in natural order has no fill: ILU(0) = LU exactly."""
    A = _tridiag(12)
    L, U = ilu.ilu0(A)
    assert np.allclose((L @ U).toarray(), A.toarray(), rtol=0, atol=1e-14)


def test_ilu0_two_by_two_and_diagonal():
    A = sp.csr_matrix(np.array([[4.0, -1.0], [-1.0, 3.0]]))
    L, U = ilu.ilu0(A)
    assert np.allclose(L.toarray(), [[1, 0], [-0.25, 1]])
    assert np.allclose(U.toarray(), [[4, -1], [0, 3 - 0.25]])
    D = sp.diags([2.0, 5.0, 7.0], format="csr")
    L, U = ilu.ilu0(D)
    assert np.allclose(U.toarray(), D.toarray()) and np.allclose(L.toarray(), np.eye(3))


def test_rb_permutation():
    perm = ilu.rb_permutation(3, 2, 2)
    i, j, k = perm % 3, (perm // 3) % 2, perm // 6
    par = (i + j + k) % 2
    nred = int(np.sum(par == 0))
    assert np.all(par[:nred] == 0) and np.all(par[nred:] == 1)
    assert np.all(np.diff(perm[:nred]) > 0) and np.all(np.diff(perm[nred:]) > 0)


def _rb_system(seed=3):
    p = random_problem(seed, 7, 6, 5, (3, 3, 2), sigma=1.0)
    A_T, A, q, _ = tpfa.build(p)
    f = ilu.RBILU0(A, p.nx, p.ny, p.nz)
    Ap = sp.csr_matrix(A)[f.perm][:, f.perm]
    return p, A, Ap, f


def test_rb_ilu0_defining_property_and_patterns():
    p, A, Ap, f = _rb_system()
    pat = (abs(Ap) > 0).astype(float)
    LU = (f.L @ f.U).tocsr()
    assert abs((LU - Ap).multiply(pat)).max() <= 1e-13 * abs(Ap).max()
    Lp = (abs(sp.tril(f.L, -1)) > 0).astype(int)
    Up = (abs(sp.triu(f.U, 1)) > 0).astype(int)
    assert (Lp - Lp.multiply(pat)).nnz == 0 and (Up - Up.multiply(pat)).nnz == 0
    assert np.all(f.L.diagonal() == 1.0)


def test_rb_ilu0_closed_form():
    """Red cells couple only to black ones: U_rr = a_rr, L_br = a_br / a_rr and the
    black pivots are a_bb - sum_r a_br a_rb / a_rr (the Schur diagonal, fill dropped)."""
    p, A, Ap, f = _rb_system(5)
    N = p.N
    nred = int(np.sum(((f.perm % p.nx) + (f.perm // p.nx) % p.ny + f.perm // (p.nx * p.ny)) % 2 == 0))
    Ad = Ap.toarray()
    U, L = f.U.toarray(), f.L.toarray()
    assert np.allclose(np.diag(U)[:nred], np.diag(Ad)[:nred], rtol=0, atol=0)
    Dr = np.diag(Ad)[:nred]
    assert np.allclose(L[nred:, :nred], Ad[nred:, :nred] / Dr[None, :], rtol=1e-15, atol=0)
    S = np.diag(Ad)[nred:] - np.einsum("br,rb->b", Ad[nred:, :nred] / Dr[None, :], Ad[:nred, nred:])
    assert np.allclose(np.diag(U)[nred:], S, rtol=1e-14)
    assert np.allclose(U[nred:, nred:], np.diag(np.diag(U)[nred:]))  # no black-black fill
    assert np.allclose(U[:nred, nred:], Ad[:nred, nred:])


def test_ilu0_smoothing_contracts_in_energy_norm():
    p, A, Ap, f = _rb_system(7)
    rng = np.random.default_rng(0)
    xs = rng.standard_normal(p.N)
    b = A @ xs
    x = np.zeros(p.N)
    e0 = x - xs
    x1 = ilu.smooth(A, b, x, f, 1)
    e1 = x1 - xs
    assert e1 @ (A @ e1) < e0 @ (A @ e0)


def test_ilu0_zero_pivot():
    with pytest.raises(ZeroDivisionError):
        ilu.ilu0(sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 1.0]])))


def test_ilu0_smoother_cuts_iterations():
    """PAPER.md:408's ILU(0) against the Jacobi stand-in: fewer cycles (config-2 recipe)."""
    base = dict(shape=(12, 22, 20), max_sweeps=100, max_iter=20000)
    rj = opl.run(make_problem(2, **base))
    ri = opl.run(make_problem(2, smoother="ilu0", **base))
    assert rj["sol"]["converged"] and ri["sol"]["converged"]
    assert ri["sol"]["iters"] < rj["sol"]["iters"] / 2
