"""Pins of the NEXT-4 oracle (oracle/cpr.py): the compressible two-phase residual and its
Jacobian, the IMPES / quasi-IMPES weights and the premultiplication
(PAPER.md:163-202), the coupled red-black ILU(0) and the two-stage preconditioner
(SPEC.md:293-354).  CPU only."""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import cpr
from oracle import fgmres as ofg
from oracle import pipeline as opl
from oracle import tpfa
from oracle.cycle import Level
from synth.configs import cpr_state, make_problem, random_problem

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cpr_hand_examples.json")


def _two_cells():
    prob = random_problem(0, 2, 1, 1, (1, 1, 1))
    prob.kx = np.ones(2)
    prob.ky = np.ones(2)
    prob.kz = np.ones(2)
    fl = cpr.Fluid(mu_w=1.0, mu_o=5.0, rho_w=1.0, rho_o=1.0, c_w=0.0, c_o=0.0, c_r=0.0,
                   phi=0.2, dt=1.0)
    return prob, fl


def _system(shape=(10, 12, 4), seed=3, fl=None, block=(5, 4, 2)):
    prob = make_problem(2, shape=shape, block=block)
    st = cpr_state(prob, seed=seed)
    fl = fl or cpr.Fluid()
    tr = tpfa.transmissibilities(prob)
    J = cpr.jacobian(fl, prob, tr, st.p, st.S, st.p_n, st.S_n, st.well_cells, st.well_rates)
    F = np.concatenate(cpr.residual(fl, prob, tr, st.p, st.S, st.p_n, st.S_n, st.well_cells,
                                    st.well_rates))
    return prob, st, fl, tr, J, F


@pytest.mark.parametrize("case", json.load(open(GOLD))["cases"], ids=lambda c: c["name"])
def test_hand_worked_two_cell_residual(case):
    prob, fl = _two_cells()
    tr = tpfa.transmissibilities(prob)
    assert np.allclose(tr[0][2], [1.0])  # T = 1 (setup line of the fixture)
    wells = case["wells"]
    wc = np.array([w[0] for w in wells], dtype=np.int64)
    wr = np.array([w[1] for w in wells], dtype=np.float64)
    a = {k: np.array(case[k], dtype=np.float64) for k in ("p", "S", "p_n", "S_n")}
    Fw, Fo = cpr.residual(fl, prob, tr, a["p"], a["S"], a["p_n"], a["S_n"], wc, wr)
    assert np.allclose(Fw, case["Fw"], rtol=0, atol=1e-15)
    assert np.allclose(Fo, case["Fo"], rtol=0, atol=1e-15)
    if "dFw0_dp0" in case:
        J = cpr.jacobian(fl, prob, tr, a["p"], a["S"], a["p_n"], a["S_n"], wc, wr)
        assert J[0, 0] == pytest.approx(case["dFw0_dp0"], abs=1e-15)
        assert J[2, 0] == pytest.approx(case["dFo0_dp0"], abs=1e-15)


def test_mass_conservation_of_fluxes():
    """Σ_i (F_β^i − A_β^i + Q_β^i) = 0: every interface flux leaves one cell and enters
    its neighbour (conservation)."""
    prob = make_problem(2, shape=(9, 7, 5), block=(3, 3, 5))
    st = cpr_state(prob, seed=5)
    fl = cpr.Fluid()
    tr = tpfa.transmissibilities(prob)
    Fw, Fo = cpr.residual(fl, prob, tr, st.p, st.S, st.p_n, st.S_n, st.well_cells[:0],
                          st.well_rates[:0])
    Aw, Ao = cpr.accumulation(fl, st.p, st.S, st.p_n, st.S_n)
    scale = np.abs(Fw - Aw).max()
    assert scale > 1.0
    assert abs(np.sum(Fw - Aw)) <= 1e-12 * scale * prob.N
    assert abs(np.sum(Fo - Ao)) <= 1e-12 * np.abs(Fo - Ao).max() * prob.N


def test_incompressible_total_equation_is_tpfa_with_total_mobility():
    """c = 0, ρ = 1: the accumulation terms of the two phases cancel in F_w + F_o and the
    flux part is (Δt/|Ω|)(A_λ p − q) with A_λ the TPFA matrix of oracle.tpfa built with the
    upstream total mobility per face (Eq. incomp-elliptic)."""
    prob = make_problem(2, shape=(8, 6, 3), block=(4, 3, 3), dx=2.0, dy=0.5, dz=3.0)
    st = cpr_state(prob, seed=2)
    fl = cpr.Fluid(rho_w=1.0, rho_o=1.0, c_w=0.0, c_o=0.0, c_r=0.0, dt=0.3)
    tr = tpfa.transmissibilities(prob)
    Fw, Fo = cpr.residual(fl, prob, tr, st.p, st.S, st.p_n, st.S_n, st.well_cells,
                          st.well_rates)
    mob = []
    for left, right, _ in tr:
        up = np.where(st.p[left] >= st.p[right], left, right)
        mob.append(cpr.mobility(fl, st.S[up], 0) + cpr.mobility(fl, st.S[up], 1))
    A_lam = tpfa.flux_matrix(prob.N, tpfa.transmissibilities(prob, mob))
    q = np.zeros(prob.N)
    np.add.at(q, st.well_cells, st.well_rates)
    vol = prob.dx * prob.dy * prob.dz
    ref = fl.dt / vol * (A_lam @ st.p - q)
    assert np.allclose(Fw + Fo, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_jacobian_matches_central_differences():
    prob, st, fl, tr, J, F = _system()
    N = prob.N
    x = np.concatenate([st.p, st.S])
    rng = np.random.default_rng(0)
    Jd = J.toarray()
    for k in rng.choice(2 * N, 24, replace=False):
        h = 1e-6 * max(1.0, abs(x[k]))
        xp, xm = x.copy(), x.copy()
        xp[k] += h
        xm[k] -= h
        Fp = np.concatenate(cpr.residual(fl, prob, tr, xp[:N], xp[N:], st.p_n, st.S_n,
                                         st.well_cells, st.well_rates))
        Fm = np.concatenate(cpr.residual(fl, prob, tr, xm[:N], xm[N:], st.p_n, st.S_n,
                                         st.well_cells, st.well_rates))
        fd = (Fp - Fm) / (2 * h)
        assert np.max(np.abs(fd - Jd[:, k])) <= 1e-7 * np.max(np.abs(Jd[:, k])), k


def test_jacobian_pattern_is_the_block_seven_point_stencil():
    prob, st, fl, tr, J, F = _system(shape=(5, 4, 3), block=(5, 4, 3))
    N = prob.N
    A_T = tpfa.flux_matrix(N, tr)
    pat = (abs(A_T) + sp.identity(N)).tocsr()
    pat.data[:] = 1
    for b in range(2):
        for v in range(2):
            blk = J[b * N:(b + 1) * N, v * N:(v + 1) * N].tocsr()
            assert blk.nnz == pat.nnz  # explicit zeros kept: every stencil entry stored
            assert (abs(blk).astype(bool) > pat.astype(bool)).nnz == 0


def test_elliptic_limit_is_symmetric():
    """Incompressible, linear relperms, equal viscosities: J*_pp with IMPES weights is the
    symmetric (Δt/|Ω|) A_T / (2 μ) (derived from Eq. incomp-elliptic)."""
    fl = cpr.Fluid(rho_w=1.0, rho_o=1.0, c_w=0.0, c_o=0.0, c_r=0.0, mu_w=2.0, mu_o=2.0,
                   nrel=1, dt=0.1)
    prob, st, fl, tr, J, F = _system(fl=fl)
    N = prob.N
    w = cpr.impes_weights(fl, st.p, st.S, st.p_n, st.S_n)
    assert np.allclose(w, 0.5, rtol=0, atol=1e-15)
    Js, _ = cpr.premultiply(J, F, w)
    Jpp = Js[:N, :N].toarray()
    assert np.max(np.abs(Jpp - Jpp.T)) <= 1e-10 * np.max(np.abs(Jpp))
    ref = fl.dt / (prob.dx * prob.dy * prob.dz) * tpfa.flux_matrix(N, tr).toarray() / (2 * 2.0)
    assert np.max(np.abs(Jpp - ref)) <= 1e-12 * np.max(np.abs(ref))


# ----------------------------------------------------------------------------- weights


@pytest.mark.parametrize("m,w", [((1.0, -1.0), (0.5, 0.5)), ((0.0, 0.0), (1.0, 0.0)),
                                 ((0.0, 3.0), (1.0, 0.0)), ((2.0, -6.0), (0.75, 0.25))])
def test_weight_system_examples(m, w):
    """SPEC.md:311-314 worked examples (the last solved by hand: 2 w1 − 6 w2 = 0,
    w1 + w2 = 1)."""
    out = cpr.weights([m[0]], [m[1]])
    assert np.allclose(out[:, 0], w, rtol=0, atol=1e-15)


def test_singular_weight_system_is_an_error():
    with pytest.raises(ZeroDivisionError):
        cpr.weights([2.0], [2.0])


def test_impes_weights_closed_form_and_cancellation():
    """∂A_w/∂S = φ ρ_w, ∂A_o/∂S = −φ ρ_o, so w = (ρ_o, ρ_w)/(ρ_w + ρ_o) at the new
    pressure; W cancels the accumulation's saturation derivative."""
    prob, st, fl, tr, J, F = _system()
    w = cpr.impes_weights(fl, st.p, st.S, st.p_n, st.S_n)
    rw, ro = cpr.density(fl, st.p, 0), cpr.density(fl, st.p, 1)
    assert np.allclose(w[0], ro / (rw + ro), rtol=1e-14)
    assert np.allclose(w[1], rw / (rw + ro), rtol=1e-14)
    assert np.allclose(w.sum(axis=0), 1.0, rtol=0, atol=1e-14)
    mw, mo = cpr.accumulation_saturation_derivative(fl, st.p, st.S, st.p_n, st.S_n)
    assert np.max(np.abs(w[0] * mw + w[1] * mo)) <= 1e-10 * np.max(np.abs(mw))


def test_quasi_impes_cancels_the_diagonal_coupling():
    """diag(J*_ps) = 0 for quasi-IMPES."""
    prob, st, fl, tr, J, F = _system()
    N = prob.N
    w = cpr.quasi_impes_weights(J, N)
    assert np.allclose(w.sum(axis=0), 1.0, rtol=0, atol=1e-14)
    Js, _ = cpr.premultiply(J, F, w)
    d = np.arange(N)
    before = np.abs(np.asarray(J[d, N + d]).ravel()).max()
    after = np.abs(np.asarray(Js[d, N + d]).ravel()).max()
    assert after <= 1e-10 * before


def test_premultiply_identity_and_second_row_and_equivalence():
    prob, st, fl, tr, J, F = _system(shape=(6, 5, 3), block=(3, 5, 3))
    N = prob.N
    Js, Fs = cpr.premultiply(J, F, np.vstack([np.ones(N), np.zeros(N)]))
    assert (Js != J).nnz == 0 and np.array_equal(Fs, F)
    w = cpr.quasi_impes_weights(J, N)
    Js, Fs = cpr.premultiply(J, F, w)
    assert (Js[N:] != J[N:]).nnz == 0 and np.array_equal(Fs[N:], F[N:])
    assert Js.nnz == J.nnz  # the block stencil pattern survives exact cancellation (C4)
    dx = np.linalg.solve(J.toarray(), -F)
    dxs = np.linalg.solve(Js.toarray(), -Fs)
    assert np.max(np.abs(dx - dxs)) <= 1e-9 * np.max(np.abs(dx))


# ----------------------------------------------------------------------------- ILU(0), CPR


def test_coupled_ilu0_reproduces_the_matrix_on_its_pattern():
    """(L U)_ij = J*_ij for (i, j) in the pattern (the defining property of ILU(0))."""
    prob, st, fl, tr, J, F = _system(shape=(6, 5, 3), block=(3, 5, 3))
    w = cpr.impes_weights(fl, st.p, st.S, st.p_n, st.S_n)
    Js, _ = cpr.premultiply(J, F, w)
    L, U, q = cpr.block_rb_ilu0(Js, prob.nx, prob.ny, prob.nz)
    Jp = Js.tocsr()[q][:, q].tocoo()
    LU = (L @ U).tocsr()
    got = np.asarray(LU[Jp.row, Jp.col]).ravel()
    assert np.max(np.abs(got - Jp.data)) <= 1e-12 * np.max(np.abs(Jp.data))


def _cpr(prob, Js, n_cycles=1, **kw):
    N = prob.N
    A_T = tpfa.flux_matrix(N, tpfa.transmissibilities(prob))
    cart = opl.cartesian_level(prob, A_T)
    lev = Level(cart["P"].matrix(), Js[:N, :N])
    return cpr.CPR(Js, N, [lev], prob.nx, prob.ny, prob.nz, n_cycles=n_cycles, **kw)


def test_cpr_zero_and_linearity():
    prob, st, fl, tr, J, F = _system()
    w = cpr.quasi_impes_weights(J, prob.N)
    Js, _ = cpr.premultiply(J, F, w)
    C = _cpr(prob, Js, n_cycles=2)
    assert np.array_equal(C.apply(np.zeros(2 * prob.N)), np.zeros(2 * prob.N))
    rng = np.random.default_rng(1)
    r1, r2 = rng.standard_normal(2 * prob.N), rng.standard_normal(2 * prob.N)
    lhs = C.apply(2.5 * r1 - 0.75 * r2)
    rhs = 2.5 * C.apply(r1) - 0.75 * C.apply(r2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))


def test_cpr_exact_on_a_decoupled_system():
    """J*_ps = 0, J_sp = 0, J_ss diagonal, exact pressure solver: the two stages together
    solve J* Δx = r exactly."""
    prob, st, fl, tr, J, F = _system(shape=(6, 5, 3), block=(3, 5, 3))
    N = prob.N
    Jd = J.tolil()
    Jd[:N, N:] = J[:N, N:].multiply(0.0)
    Jd[N:, :N] = J[N:, :N].multiply(0.0)
    Jss = J[N:, N:].tolil()
    off = Jss - sp.diags(Jss.diagonal())
    Jd[N:, N:] = Jss - off.multiply(1.0)
    Js = Jd.tocsr()
    Jpp = Js[:N, :N].tocsc()
    C = _cpr(prob, Js, pressure_solve=lambda r: spla.spsolve(Jpp, r))
    r = np.random.default_rng(2).standard_normal(2 * N)
    dx = C.apply(r)
    ref = spla.spsolve(Js.tocsc(), r)
    assert np.max(np.abs(dx - ref)) <= 1e-9 * np.max(np.abs(ref))


def test_cpr_gmres_beats_ilu0_alone():
    """GMRES right-preconditioned by the two-stage CPR needs fewer iterations to 1e-8 than
    GMRES with ILU(0) alone (derived: comparative run)."""
    prob, st, fl, tr, J, F = _system(shape=(16, 20, 6), block=(4, 5, 3))
    N = prob.N
    w = cpr.impes_weights(fl, st.p, st.S, st.p_n, st.S_n)
    Js, Fs = cpr.premultiply(J, F, w)
    C = _cpr(prob, Js)
    o1 = ofg.fgmres(Js, -Fs, np.zeros(2 * N), [], tol=1e-8, restart=40, max_iter=200,
                    precond=C.apply)
    o2 = ofg.fgmres(Js, -Fs, np.zeros(2 * N), [], tol=1e-8, restart=40, max_iter=200,
                    precond=C.corrector)
    assert o1["converged"]
    assert o1["iters"] < o2["iters"]
