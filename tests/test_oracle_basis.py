"""Oracle pins — MsRSB smoothing (O6–O7).

* B1 hand-derived sweeps on a 4-cell chain (tests/golden/basis_1d_hand.json).
* B2 closed form: uniform K, odd block sizes, converged basis = tensor-product
  hat (Q1 interpolation between block-centre cells, constant beyond the
  outermost centres) — SURVEY.md §8.c pins table.
* B3 invariants: partition of unity, 0 <= P <= 1, zero outside the
  pattern, P = 1 on single-support cells, M = 1 gives ones, no
  leakage past a sealing fault, locality (n sweeps reach graph
  distance n), stationarity of the converged fixed point.
"""
import json
import os

import numpy as np
import pytest

from oracle import basis, partition, support, tpfa
from synth.configs import Problem, make_problem, random_problem

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _level(p):
    A_T, A, q, _ = tpfa.build(p)
    part, M, _ = partition.cartesian(p.nx, p.ny, p.nz, p.block)
    pat = support.box_pattern(p.nx, p.ny, p.nz, p.block)
    return A_T, part, M, pat, basis.indicator(part, pat)


def test_hand_sweeps_1d():
    g = json.load(open(os.path.join(GOLD, "basis_1d_hand.json")))
    for case in g["cases"]:
        k = np.array(case["K"])
        p = Problem("h", 4, 1, 1, k, k, k, np.array([0]), np.array([0.0]), (2, 1, 1))
        A_T, part, M, pat, P0 = _level(p)
        assert np.allclose(tpfa.transmissibilities(p)[0][2], case["T_faces"], rtol=1e-15)
        P1, d1 = basis.sweep(P0, A_T, 2.0 / 3.0)
        assert np.allclose(P1.dense(), np.array(case["P1"]), rtol=0, atol=1e-15)
        assert abs(d1 - case["delta1"]) < 1e-15
        if "P2" in case:
            P2, _ = basis.sweep(P1, A_T, 2.0 / 3.0)
            assert np.allclose(P2.dense(), np.array(case["P2"]), rtol=0, atol=1e-15)


def _hat(n, b):
    nb = -(-n // b)
    c = np.arange(nb) * b + (b - 1) / 2.0
    H = np.zeros((n, nb))
    x = np.arange(n)
    for J in range(nb):
        v = np.maximum(0.0, 1.0 - np.abs(x - c[J]) / b)
        if J == 0:
            v[x <= c[0]] = 1.0
        if J == nb - 1:
            v[x >= c[-1]] = 1.0
        H[:, J] = v
    return H


@pytest.mark.parametrize("dims", [(25, 25, 1, (5, 5, 1)), (21, 10, 1, (7, 5, 1)),
                                  (15, 15, 15, (5, 5, 5))])
def test_hat_closed_form_odd_blocks(dims):
    nx, ny, nz, blk = dims
    k = np.ones(nx * ny * nz)
    p = Problem("u", nx, ny, nz, k, k, k, np.array([0]), np.array([0.0]), blk)
    A_T, part, M, pat, P0 = _level(p)
    P, n, d = basis.smooth(P0, A_T, 2.0 / 3.0, 20000, 1e-15)
    assert d[-1] <= 1e-15
    H = np.kron(_hat(nz, blk[2]), np.kron(_hat(ny, blk[1]), _hat(nx, blk[0])))
    assert np.abs(P.dense() - H).max() < 1e-12


def test_even_block_interior_alpha():
    """1D even blocks: interior ramp starts near α with (n-1)α² - (n+1)α + 1 = 0
    (approximate on finite chains, 1e-2)."""
    n_cells, b = 96, 8
    k = np.ones(n_cells)
    p = Problem("e", n_cells, 1, 1, k, k, k, np.array([0]), np.array([0.0]), (b, 1, 1))
    A_T, part, M, pat, P0 = _level(p)
    P, _, _ = basis.smooth(P0, A_T, 2.0 / 3.0, 50000, 1e-15)
    alpha = ((b + 1) - np.sqrt((b + 1) ** 2 - 4 * (b - 1))) / (2 * (b - 1))
    D = P.dense()
    J = 6                                    # interior block
    x_first = J * b - b // 2                 # first cell of S_J's left half (past C(J-1))
    assert abs(D[x_first, J] - alpha) < 1e-2


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_invariants_heterogeneous(seed):
    p = random_problem(seed, 13, 11, 6, (4, 3, 3), sigma=2.0)
    A_T, part, M, pat, P0 = _level(p)
    P = P0
    for n in range(1, 25):
        P, d = basis.sweep(P, A_T, 2.0 / 3.0)
        rs = np.bincount(P.rows, weights=P.vals, minlength=p.N)
        assert np.max(np.abs(rs - 1.0)) <= 1e-14
        assert P.vals.min() >= 0.0 and P.vals.max() <= 1.0
    single = np.diff(pat.indptr) == 1
    assert np.all(P.vals[np.repeat(single, np.diff(pat.indptr))] == 1.0)


def test_single_block_ones():
    p = random_problem(5, 7, 6, 1, (7, 6, 1))
    A_T, part, M, pat, P0 = _level(p)
    assert M == 1
    P, n, d = basis.smooth(P0, A_T, 2.0 / 3.0, 10, 0.0, fixed=True)
    assert np.all(P.vals == 1.0) and np.all(d == 0.0)


def test_locality_n_sweeps():
    """After n sweeps P_ij = 0 exactly for cells at graph distance > n from Ω_j."""
    p = random_problem(6, 20, 1, 1, (5, 1, 1))
    A_T, part, M, pat, P0 = _level(p)
    P = P0
    for n in range(1, 4):
        P, _ = basis.sweep(P, A_T, 2.0 / 3.0)
        D = P.dense()
        for J in range(M):
            cells = np.nonzero(part == J)[0]
            dist = np.min(np.abs(np.arange(20)[:, None] - cells[None, :]), axis=1)
            assert np.all(D[dist > n, J] == 0.0)
            assert np.all(D[(dist <= n) & (np.asarray(pat[:, J].todense()).ravel() > 0), J] > 0)


def test_no_leak_past_sealing_fault():
    """a sealing plane inside a support stops the basis exactly."""
    faults = [("x", 7, 0, 6, 0.0)]                 # full plane between i=7 and i=8
    p = random_problem(8, 16, 6, 1, (4, 6, 1), faults=faults)
    A_T, part, M, pat, P0 = _level(p)
    P, _, _ = basis.smooth(P0, A_T, 2.0 / 3.0, 200, 0.0, fixed=True)
    D = P.dense()
    i = np.arange(p.N) % p.nx
    # block J=1 covers i=4..7 (left of the fault): its support reaches i=9 but stays 0 there
    assert np.all(D[i >= 8, 1] == 0.0)
    assert np.all(D[i <= 7, 2] == 0.0)
    assert np.max(np.abs(D.sum(axis=1) - 1.0)) < 1e-14


def test_converged_stationarity():
    """Fixed point of A5+A6: with Q = A_T P restricted to the pattern,
    Q_ij = P_ij Σ_k Q_ik for every pattern entry (from P = N(P - ω D^-1 Q))."""
    p = random_problem(9, 12, 10, 1, (4, 5, 1), sigma=1.0)
    A_T, part, M, pat, P0 = _level(p)
    P, n, d = basis.smooth(P0, A_T, 2.0 / 3.0, 40000, 1e-15)
    D = P.dense()
    AP = A_T @ D
    mask = pat.toarray() > 0
    lhs = AP[mask]
    rhs = (D * (AP * mask).sum(axis=1, keepdims=True))[mask]
    assert np.max(np.abs(lhs - rhs)) < 1e-11 * np.max(np.abs(AP))


def test_zero_diagonal_rejected():
    k = np.ones(1)
    p = Problem("one", 1, 1, 1, k, k, k, np.array([0]), np.array([0.0]), (1, 1, 1))
    A_T, part, M, pat, P0 = _level(p)
    with pytest.raises(ValueError):
        basis.sweep(P0, A_T, 2.0 / 3.0)
