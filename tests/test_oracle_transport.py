"""Oracle pins — config-4 transport and the sequential outer loop (O12).

Closed forms of the quadratic-relperm fractional flow (BASELINE.json configs[3]);
the exact first sub-step from S = 0 (only injector cells gain water: h q/(φ|Ω|));
water mass balance of a single sub-step (interior face fluxes cancel, PAPER.md:39
"mass-conservative"); the discrete maximum principle 0 <= S <= 1 under the CFL
sub-step rule (reading A18); a hand-worked 3-cell chain; upstream mobility for
uniform saturation and ties (reading A17); and that the outer loop's pressure step
matches the direct sparse solve.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import tpfa, transport
from oracle.grid import all_faces
from synth.configs import Problem, make_problem, random_problem


def test_fractional_flow_closed_forms():
    f = transport.fractional_flow
    assert f(0.0, 1.0, 5.0) == 0.0 and f(1.0, 1.0, 5.0) == 1.0
    assert abs(f(0.5, 1.0, 5.0) - 5.0 / 6.0) < 1e-15          # 0.25 / (0.25 + 0.05)
    assert abs(f(0.5, 2.0, 2.0) - 0.5) < 1e-15                 # equal viscosities
    assert transport.total_mobility(0.0, 1.0, 5.0) == 0.2      # 1/μ_o
    assert transport.total_mobility(1.0, 1.0, 5.0) == 1.0      # 1/μ_w
    # forward-difference slope maximum vs the analytic derivative on a fine grid
    s = np.linspace(0, 1, 200001)
    lw, lo = s * s, (1 - s) ** 2 / 5.0
    dfw = (2 * s * lo + 2 * (1 - s) / 5.0 * lw) / (lw + lo) ** 2
    assert abs(transport.fw_slope_max(1.0, 5.0) - dfw.max()) < 2e-2 * dfw.max()


def _setup(prob):
    A_T, A, q, trans = tpfa.build(prob)
    p = spla.spsolve(A.tocsc(), q)
    phi = np.full(prob.N, prob.phi)
    return trans, p, phi, q


def test_first_substep_from_dry_reservoir_exact():
    prob = random_problem(3, 9, 8, 4, (3, 4, 2), sigma=1.0)
    trans, p, phi, q = _setup(prob)
    h = 1e-4  # well inside the CFL limit: one sub-step
    fl = transport.face_fluxes(trans, p)
    assert transport.cfl_substeps(fl, q, phi, 1.0, h, 1.0, 5.0) == 1
    S, n = transport.transport(trans, p, np.zeros(prob.N), phi, q, 1.0, 1.0, 5.0, h)
    assert n == 1
    expect = np.where(q > 0, h * q / phi, 0.0)
    assert np.array_equal(S, expect)


def test_single_substep_mass_balance():
    prob = random_problem(4, 10, 7, 5, (5, 7, 5), sigma=1.5)
    trans, p, phi, q = _setup(prob)
    rng = np.random.default_rng(0)
    S0 = rng.uniform(0.0, 0.8, prob.N)
    h = 1e-5
    S1, n = transport.transport(trans, p, S0, phi, q, 1.0, 1.0, 5.0, h)
    assert n == 1
    fw = transport.fractional_flow(S0, 1.0, 5.0)
    produced = np.sum(np.where(q < 0, -q * fw, 0.0))
    injected = np.sum(np.where(q > 0, q, 0.0))
    lhs = np.sum(phi * (S1 - S0))
    # rounding of S1 = S0 + ΔS (|S| < 1) is the only error: <= N ε max φ
    assert abs(lhs - h * (injected - produced)) <= prob.N * np.finfo(float).eps * phi.max()


def test_maximum_principle_over_steps():
    prob = random_problem(5, 12, 10, 3, (4, 5, 3), sigma=2.0)
    trans, p, phi, q = _setup(prob)
    dt = transport.step_size(prob, q, phi, 0.05)
    S = np.zeros(prob.N)
    for _ in range(6):
        S, n = transport.transport(trans, p, S, phi, q, 1.0, 1.0, 5.0, dt)
        assert n >= 1
        assert S.min() >= -1e-15 and S.max() <= 1.0 + 1e-15


def test_three_cell_chain_by_hand():
    # cells 0-1-2 along x, T = 1 (K = 1), p = [2, 1, 0], q = [+1, 0, -1], φ = 1/2
    prob = Problem("chain", 3, 1, 1, np.ones(3), np.ones(3), np.ones(3),
                   np.array([0, 2]), np.array([1.0, -1.0]), (1, 1, 1), phi=0.5)
    A_T, A, q, trans = tpfa.build(prob)
    p = np.array([2.0, 1.0, 0.0])
    S0 = np.array([0.5, 0.0, 0.0])
    h = 0.01
    S1, n = transport.transport(trans, p, S0, np.full(3, 0.5), q, 1.0, 1.0, 5.0, h)
    f = 5.0 / 6.0                        # f_w(0.5)
    # cell 0: +1 injected, -F f_w(S_0) out (F = 1); cell 1: +F f_w(S_0) in, 0 out; cell 2: 0
    assert n == 1
    assert np.allclose(S1, [0.5 + h / 0.5 * (1.0 - f), h / 0.5 * f, 0.0], rtol=0, atol=1e-16)


def test_upstream_mobility_uniform_and_ties():
    prob = random_problem(6, 5, 4, 3, (5, 4, 3))
    faces = all_faces(prob.nx, prob.ny, prob.nz)
    rng = np.random.default_rng(1)
    p = rng.standard_normal(prob.N)
    mob = transport.upstream_mobility(faces, p, np.full(prob.N, 0.3), 1.0, 5.0)
    lam = transport.total_mobility(0.3, 1.0, 5.0)
    assert all(np.all(m == lam) for m in mob)
    S = np.arange(prob.N) / prob.N
    mob = transport.upstream_mobility(faces, np.zeros(prob.N), S, 1.0, 5.0)  # all ties
    for (left, _), m in zip(faces, mob):
        assert np.array_equal(m, transport.total_mobility(S[left], 1.0, 5.0))


def test_outer_loop_pressure_matches_direct_solve():
    prob = make_problem(4, shape=(12, 22, 10), max_sweeps=20, cycle_tol=1e-10, max_iter=20000)
    out = transport.run(prob, steps=3, k_adapt=5, pv_per_step=0.02)
    assert len(out["steps"]) == 3
    # rebuild step 3's operator from step 2's saturation/pressure and solve directly
    faces = all_faces(prob.nx, prob.ny, prob.nz)
    s2 = out["steps"][1]
    mob = transport.upstream_mobility(faces, s2["p"], s2["S"], 1.0, 5.0)
    A_T, A, q, _ = tpfa.build(prob, mob)
    p_direct = spla.spsolve(A.tocsc(), q)
    p3 = out["steps"][2]["p"]
    assert np.linalg.norm(p3 - p_direct) <= 1e-6 * np.linalg.norm(p_direct)
    for r in out["steps"]:
        assert r["converged"] and 0 <= r["S"].min() and r["S"].max() <= 1.0
