"""Oracle pins — Galerkin coarse operator, coarse solve, and the cycle (O8–O11).

RAP: symmetry, A_c·1 = 0 for the zero-row-sum A_T, P = I gives
A_c = A, 2-block constant basis gives [[T,-T],[-T,T]]
(SPEC.md:454).  LU: SPEC.md:84 example and the singular case.
Cycle: zero residual leaves x unchanged; identity partition exact
in one cycle; range(P) exactness of the Galerkin correction;
linearity in the residual; converged pressure vs direct sparse
solve; line-drive closed form; dynamic stage reduces iterations (PAPER.md:274,
:333 qualitative claim).  Cost model Eq. (9).
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import basis, coarse, cost, cycle, partition, pipeline, support, tpfa
from synth.configs import Problem, make_problem, random_problem

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _smoothed(p, sweeps=30):
    A_T, A, q, _ = tpfa.build(p)
    part, M, _ = partition.cartesian(p.nx, p.ny, p.nz, p.block)
    pat = support.box_pattern(p.nx, p.ny, p.nz, p.block)
    P, _, _ = basis.smooth(basis.indicator(part, pat), A_T, 2.0 / 3.0, sweeps, 0.0, fixed=True)
    return A_T, A, q, P.matrix(), M


def test_rap_invariants():
    p = random_problem(1, 12, 9, 5, (4, 3, 5), sigma=1.5)
    A_T, A, q, P, M = _smoothed(p)
    AcT = coarse.galerkin(P, A_T)
    assert np.allclose(AcT, AcT.T, rtol=0, atol=1e-13 * np.abs(AcT).max())
    assert np.max(np.abs(AcT @ np.ones(M))) < 1e-12 * np.abs(AcT).max()
    Ac = coarse.galerkin(P, A)
    w = np.linalg.eigvalsh(0.5 * (Ac + Ac.T))
    assert w.min() > 0                                             # SPD with the gauge


def test_rap_identity_and_two_block():
    p = random_problem(2, 6, 1, 1, (1, 1, 1))
    A_T, A, q, _ = tpfa.build(p)
    assert np.allclose(coarse.galerkin(sp.identity(6, format="csr"), A), A.toarray(), rtol=0,
                       atol=0)
    P = cycle.constant_basis(np.array([0, 0, 0, 1, 1, 1]), 2)
    Ac = coarse.galerkin(P, A_T)
    T = tpfa.transmissibilities(p)[0][2][2]                        # face between cells 2|3
    assert np.allclose(Ac, [[T, -T], [-T, T]], rtol=1e-14, atol=0)


def test_lu_examples():
    s = coarse.CoarseSolver(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert np.allclose(s.solve(np.array([3.0, 3.0])), [1.0, 1.0], rtol=0, atol=1e-15)
    with pytest.raises(coarse.SingularCoarse):
        coarse.CoarseSolver(np.array([[1.0, 1.0], [1.0, 1.0]]))


def test_coarse_residual_bound():
    rng = np.random.default_rng(0)
    B = rng.standard_normal((50, 50))
    Ac = B @ B.T + 50 * np.eye(50)
    b = rng.standard_normal(50)
    x = coarse.CoarseSolver(Ac).solve(b)
    assert np.max(np.abs(Ac @ x - b)) <= 1e-10 * np.max(np.abs(b))


def _levels(p, sweeps=30):
    A_T, A, q, P, M = _smoothed(p, sweeps)
    return A, q, [cycle.Level(P, A)]


def test_zero_residual_unchanged():
    p = random_problem(3, 10, 8, 1, (5, 4, 1))
    A, q, levels = _levels(p)
    x = np.random.default_rng(1).standard_normal(p.N)
    b = A @ x
    x1 = cycle.stage(A, A.diagonal(), b, x, levels[0], 2.0 / 3.0, 1, False)
    assert np.max(np.abs(x1 - x)) < 1e-13 * np.max(np.abs(x))


def test_identity_partition_exact_one_cycle():
    p = random_problem(4, 6, 5, 1, (1, 1, 1))
    A_T, A, q, _ = tpfa.build(p)
    lev = cycle.Level(sp.identity(p.N, format="csr"), A)
    out = cycle.iterate(A, q, np.zeros(p.N), [lev], tol=1e-12, max_iter=5)
    assert out["iters"] == 1 and out["res"][-1] < 1e-13


def test_range_of_P_exact():
    """ν = 0, x0 = 0, b = A P y  ⇒  one coarse correction returns P y exactly."""
    p = random_problem(5, 12, 10, 1, (4, 5, 1), sigma=1.0)
    A, q, levels = _levels(p)
    P = levels[0].P
    y = np.random.default_rng(2).standard_normal(P.shape[1])
    b = A @ (P @ y)
    x = cycle.stage(A, A.diagonal(), b, np.zeros(p.N), levels[0], 2.0 / 3.0, 0, False)
    assert np.max(np.abs(x - P @ y)) < 1e-10 * np.max(np.abs(P @ y))


def test_cycle_linear_in_residual():
    p = random_problem(6, 10, 9, 3, (5, 3, 3))
    A, q, levels = _levels(p)
    rng = np.random.default_rng(3)
    r1, r2 = rng.standard_normal(p.N), rng.standard_normal(p.N)
    z = np.zeros(p.N)
    f = lambda r: cycle.stage(A, A.diagonal(), r, z, levels[0], 2.0 / 3.0, 1, False)
    lhs = f(2.0 * r1 - 3.0 * r2)
    rhs = 2.0 * f(r1) - 3.0 * f(r2)
    assert np.max(np.abs(lhs - rhs)) < 1e-12 * np.max(np.abs(lhs))


@pytest.mark.parametrize("post", [False, True])
def test_converges_to_direct_solve(post):
    p = make_problem(1, shape=(32, 32), block=(8, 8, 1), post_smooth=post)
    r = pipeline.run(p, sweeps=100)
    xe = spla.spsolve(r["A"].tocsc(), r["q"])
    s = r["sol"]
    assert s["converged"] and s["res"][-1] <= 1e-6
    assert np.linalg.norm(r["A"] @ s["x"] - r["q"]) <= 1e-6 * np.linalg.norm(r["q"]) * 1.0000001
    assert np.linalg.norm(s["x"] - xe) / np.linalg.norm(xe) < 1e-3


def test_line_drive_closed_form():
    """Uniform K; source plane x=0 (+q per cell), sink plane x=nx-1 (-q per cell):
    exact TPFA pressure p(x) = -x q / T (gauge p_0 = 0)."""
    nx, ny, nz = 15, 7, 5
    N = nx * ny * nz
    k = np.full(N, 2.0)                         # T = 2 for unit cells
    cells = np.arange(N)
    i = cells % nx
    src = np.concatenate([cells[i == 0], cells[i == nx - 1]])
    rates = np.concatenate([np.full((i == 0).sum(), 0.5), np.full((i == nx - 1).sum(), -0.5)])
    p = Problem("ld", nx, ny, nz, k, k.copy(), k.copy(), src, rates, (5, 7, 5),
                max_sweeps=100, sweep_tol=1e-6, cycle_tol=1e-10)
    r = pipeline.run(p)
    exact = -i * 0.5 / 2.0
    assert r["sol"]["converged"]
    assert np.max(np.abs(r["sol"]["x"] - exact)) < 1e-8


def test_dynamic_stage_helps():
    """adding the Δp-adapted constant basis reduces iterations."""
    p = make_problem(1, shape=(32, 32), block=(8, 8, 1), max_sweeps=100)
    base = pipeline.run(p)["sol"]
    p.dynamic = True
    dyn = pipeline.run(p, record_dynamic=True)["sol"]
    assert dyn["converged"] and dyn["iters"] < base["iters"]
    assert all(part is not None and part.max() + 1 == M for _, part, M in dyn["dyn"])


def test_fixed_iters_and_zero_rhs():
    p = random_problem(7, 8, 8, 1, (4, 4, 1))
    A, q, levels = _levels(p)
    out = cycle.iterate(A, np.zeros(p.N), np.zeros(p.N), levels, tol=1e-6)
    assert out["iters"] == 0 and out["converged"]
    out = cycle.iterate(A, q, np.zeros(p.N), levels, fixed_iters=7)
    assert out["iters"] == 7 and len(out["res"]) == 8


def test_cost_model_spec():
    g = json.load(open(os.path.join(GOLD, "cost_spec_examples.json")))
    for c in g["cases"]:
        assert cost.cost_per_iteration(c["N"], c["Np"], c["d"], c["b"], c["Nc"]) == c["c"]
    r = [cost.cost_per_iteration(1, 2, 15, 4, nc) / cost.cost_per_iteration(1, 1, 15, 4, nc)
         for nc in (1, 2, 3, 4)]
    assert all(a > b for a, b in zip(r, r[1:]))         # PAPER.md:430 "diminishes"


def test_dynamic_stage_wiring():
    """Pins the dynamic-stage wiring of O11 (readings A12, A14, A15):
    (i) no stage at k = 1; (ii) the k-th partition is dynamic_partition of
    x_start(k) - x_start(k-1), the update over the PREVIOUS full iteration, with both
    iterates re-run independently (fixed_iters = k-1, k-2); (iii) the stage runs after the
    static levels — the iterate after 3 iterations equals a hand-sequenced chain of
    cycle.stage() calls in that order.  An x_end(k) - x_start(k) reading, a start at k = 1,
    or the dynamic stage placed first each fail one of these."""
    p = make_problem(1, shape=(24, 24), block=(6, 6, 1), max_sweeps=40, dynamic=True)
    r = pipeline.run(p, fixed_iters=3, record_dynamic=True)
    A, q, levels = r["A"], r["q"], r["levels"]
    recs = r["sol"]["dyn"]
    assert [k for k, _, _ in recs] == [2, 3]                                     # (i)
    xs = [np.zeros(p.N)] + [pipeline.run(p, fixed_iters=k, levels_info=r["levels_info"])
                            ["sol"]["x"] for k in (1, 2)]
    for k, part, M in recs:                                                      # (ii)
        ref, Mr = partition.dynamic_partition(xs[k - 1] - xs[k - 2], p.nx, p.ny, p.nz,
                                              p.dyn_edges, p.dyn_max_blocks)
        assert Mr == M and np.array_equal(part, ref)
    DA = A.diagonal()                                                            # (iii)
    x = np.zeros(p.N)
    starts = []
    for k in (1, 2, 3):
        starts.append(x.copy())
        for lev in levels:
            x = cycle.stage(A, DA, q, x, lev, p.omega_s, p.nu, p.post_smooth)
        if k >= 2:
            part, M = partition.dynamic_partition(starts[k - 1] - starts[k - 2], p.nx, p.ny,
                                                  p.nz, p.dyn_edges, p.dyn_max_blocks)
            dl = cycle.Level(cycle.constant_basis(part, M), A)
            # the dynamic stage is built from x_start(k) but applied after the static ones
            x = cycle.stage(A, DA, q, x, dl, p.omega_s, p.nu, p.post_smooth)
    assert np.array_equal(x, r["sol"]["x"])
