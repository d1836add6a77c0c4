"""Oracle pins — TPFA (O1–O3).  SPEC.md:156-167 worked values
invariants, and the gauge closed form (reading A7)."""
import json
import os

import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import grid, tpfa
from synth.configs import Problem, random_problem

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _uniform(nx, ny, nz, K=1.0, **kw):
    n = nx * ny * nz
    k = np.full(n, K)
    return Problem("u", nx, ny, nz, k, k.copy(), k.copy(), np.array([0]), np.array([0.0]),
                   (1, 1, 1), **kw)


def test_face_counts_spec():
    g = json.load(open(os.path.join(GOLD, "tpfa_spec_examples.json")))
    for case in g["face_counts"]:
        nx, ny, nz = case["grid"]
        n = sum(len(f[0]) for f in grid.all_faces(nx, ny, nz))
        assert n == case["faces"]


def test_pair_transmissibility_spec():
    g = json.load(open(os.path.join(GOLD, "tpfa_spec_examples.json")))
    for case in g["pairs"]:
        k = np.array(case["K"])
        p = Problem("p", 2, 1, 1, k, k, k, np.array([0]), np.array([0.0]), (1, 1, 1))
        tr = tpfa.transmissibilities(p)
        assert tr[0][2][0] == case["T"]


def test_barrier_limit():
    k = np.array([1.0, 1e-300])
    p = Problem("p", 2, 1, 1, k, k, k, np.array([0]), np.array([0.0]), (1, 1, 1))
    assert tpfa.transmissibilities(p)[0][2][0] < 1e-299


def test_nonunit_cells_closed_form():
    # t = K A/(Δ/2) with A = dy*dz for x-faces: dx=2, dy=3, dz=5, K=7 → t = 7*15/1 = 105, T = 52.5
    p = _uniform(2, 2, 2, K=7.0, dx=2.0, dy=3.0, dz=5.0)
    tr = tpfa.transmissibilities(p)
    assert np.allclose(tr[0][2], 52.5, rtol=0, atol=1e-12)
    assert np.allclose(tr[1][2], 7 * 10 / 1.5 / 2, rtol=1e-15)   # A = dx*dz = 10, Δ/2 = 1.5
    assert np.allclose(tr[2][2], 7 * 6 / 2.5 / 2, rtol=1e-15)    # A = dx*dy = 6, Δ/2 = 2.5


def test_nonpositive_perm_rejected():
    p = _uniform(2, 1, 1)
    p.kx[1] = 0.0
    with pytest.raises(ValueError):
        tpfa.transmissibilities(p)


@pytest.mark.parametrize("seed", [0, 1])
def test_flux_matrix_invariants(seed):
    p = random_problem(seed, 5, 4, 3, (2, 2, 2), sigma=2.0)
    A_T, A, q, tr = tpfa.build(p)
    d = A_T.toarray()
    assert np.allclose(d, d.T, atol=0)                         # symmetric
    assert np.max(np.abs(d.sum(axis=1))) < 1e-12 * np.abs(d).max()   # zero row sums
    off = d - np.diag(np.diag(d))
    assert np.all(off <= 0) and np.all(np.diag(d) > 0)          # M-matrix sign pattern
    # swapping i,l leaves T unchanged
    k = p.kx.copy()
    p2 = random_problem(seed, 5, 4, 3, (2, 2, 2), sigma=2.0)
    p2.kx = k[::-1].copy(); p2.ky = p2.ky[::-1].copy(); p2.kz = p2.kz[::-1].copy()
    tr2 = tpfa.transmissibilities(p2)
    assert np.allclose(np.sort(tr2[0][2]), np.sort(tr[0][2]), rtol=1e-15)


def test_monotone_in_perm():
    p = random_problem(3, 4, 4, 1, (2, 2, 1))
    t0 = tpfa.transmissibilities(p)[0][2]
    p.kx[5] *= 2.0
    t1 = tpfa.transmissibilities(p)[0][2]
    assert np.all(t1 >= t0)


def test_gauge_closed_form():
    """A p = q (A = A_T with A_00 doubled) ⇔ A_T p = q and p_0 = 0 when Σq = 0 (A7)."""
    p = random_problem(4, 6, 5, 4, (2, 2, 2), sigma=1.5)
    A_T, A, q, _ = tpfa.build(p)
    assert abs(q.sum()) == 0.0
    x = spla.spsolve(A.tocsc(), q)
    assert abs(x[0]) < 1e-12 * np.abs(x).max()
    assert np.linalg.norm(A_T @ x - q) < 1e-11 * np.linalg.norm(q)
    assert A[0, 0] == 2 * A_T[0, 0]


def test_anisotropic_per_axis_closed_form():
    """Per-axis K selection (config 5 has Kz != Kx): heterogeneous kx, ky, kz fields with
    distinct values per axis give T_f = 2 K_a,i K_a,l / (K_a,i + K_a,l) * A_a / Δ_a on each
    axis from THAT axis' permeability — a kx-on-every-axis slip fails."""
    nx, ny, nz = 3, 2, 2
    n = nx * ny * nz
    c = np.arange(n)
    kx = 1.0 + c            # 1..12
    ky = 100.0 + 10.0 * c   # distinct from kx everywhere
    kz = 0.01 * (1.0 + c)
    p = Problem("a", nx, ny, nz, kx, ky, kz, np.array([0]), np.array([0.0]), (1, 1, 1),
                dx=1.0, dy=2.0, dz=4.0)
    tr = tpfa.transmissibilities(p)
    areas = (2.0 * 4.0, 1.0 * 4.0, 1.0 * 2.0)   # A_x = dy dz, A_y = dx dz, A_z = dx dy
    dists = (1.0, 2.0, 4.0)
    for a, (left, right, T) in enumerate(tr):
        K = (kx, ky, kz)[a]
        # harmonic mean of the two half-transmissibilities K A / (Δ / 2), written out
        t_l = K[left] * areas[a] / (dists[a] / 2.0)
        t_r = K[right] * areas[a] / (dists[a] / 2.0)
        expect = 1.0 / (1.0 / t_l + 1.0 / t_r)
        assert np.allclose(T, expect, rtol=1e-15, atol=0.0), a
        # and by hand for the first face of each axis
    assert np.isclose(tr[0][2][0], 1.0 / (1.0 / (1 * 8 / 0.5) + 1.0 / (2 * 8 / 0.5)))  # kx 1 | 2
    assert np.isclose(tr[1][2][0], 1.0 / (1.0 / (100 * 4 / 1.0) + 1.0 / (130 * 4 / 1.0)))  # ky 100 | 130
    assert np.isclose(tr[2][2][0], 1.0 / (1.0 / (0.01 * 2 / 2.0) + 1.0 / (0.07 * 2 / 2.0)))  # kz .01 | .07
