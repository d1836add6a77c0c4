"""Pins for the NEXT-3 oracle pieces (oracle/partition.py wells_partition,
indicator_partition; oracle/support.py dilated_pattern; general MsRSB levels).

SPEC.md:401-426 examples, brute force on tiny grids, and invariants (requirement 2,
partition of unity, no leak across a sealing face)."""
import collections
import itertools

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import basis as obasis
from oracle import partition as opart
from oracle import pipeline as opl
from oracle import support as osup
from oracle import tpfa
from synth.configs import make_problem, random_problem


# ---------------------------------------------------------------- well partition
def test_wells_five_spot_six_blocks():
    """'six coarse blocks (one for each well plus one ...)'."""
    p = make_problem(2, shape=(24, 44, 20))
    part, M = opart.wells_partition(p.nx, p.ny, p.nz, p.wells(), 2)
    assert len(p.wells()) == 5 and M == 6
    assert set(np.unique(part)) == set(range(6))


def test_wells_radius_zero_is_perforations():
    p = make_problem(2, shape=(24, 44, 20))
    part, M = opart.wells_partition(p.nx, p.ny, p.nz, p.wells(), 0)
    for w, cells in enumerate(p.wells()):
        assert np.array_equal(np.sort(np.flatnonzero(part == w)), np.sort(cells))
    assert M == 6


def test_wells_tie_goes_to_lower_index_1d():
    """overlapping radii on a 1D chain -> the midpoint joins the lower well."""
    part, M = opart.wells_partition(9, 1, 1, [np.array([2]), np.array([6])], 2)
    assert part.tolist() == [0, 0, 0, 0, 0, 1, 1, 1, 1] and M == 2
    part, M = opart.wells_partition(9, 1, 1, [np.array([6]), np.array([2])], 2)
    assert part.tolist() == [1, 1, 1, 1, 0, 0, 0, 0, 0] and M == 2  # well 0 is now on the right


def test_wells_brute_force_3d():
    rng = np.random.default_rng(3)
    nx, ny, nz = 7, 6, 5
    wells = [rng.choice(nx * ny * nz, size=int(rng.integers(1, 4)), replace=False) for _ in range(3)]
    for radius in (0, 1, 2):
        part, M = opart.wells_partition(nx, ny, nz, wells, radius)
        for c in range(nx * ny * nz):
            i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
            best, owner = None, None
            for w, cells in enumerate(wells):
                for q in cells:
                    qi, qj, qk = q % nx, (q // nx) % ny, q // (nx * ny)
                    d = max(abs(i - qi), abs(j - qj), abs(k - qk))
                    if best is None or d < best:
                        best, owner = d, w
            assert part[c] == (owner if best <= radius else len(wells))
        assert M == len(wells) + int(np.any(part == len(wells)))


def test_wells_errors():
    with pytest.raises(ValueError):
        opart.wells_partition(4, 1, 1, [np.array([9])], 1)
    with pytest.raises(ValueError):
        opart.wells_partition(4, 1, 1, [np.array([1])], -1)


# ---------------------------------------------------------------- indicator partition
def test_indicator_spec_examples():
    """SPEC.md:406-409."""
    part, M = opart.indicator_partition(np.array([0.0, 0.5, 10.0, 11.0]), 4, 1, 1, [1.0])
    assert part.tolist() == [0, 0, 1, 1] and M == 2
    part, M = opart.indicator_partition(np.full(6, 3.0), 6, 1, 1, [1.0])
    assert M == 1
    part, M = opart.indicator_partition(np.array([5.0, 0.0, 5.0]), 3, 1, 1, [1.0])
    assert part.tolist() == [0, 1, 2] and M == 3


def _bfs_components(bins, nx, ny, nz):
    N = nx * ny * nz
    lab = -np.ones(N, dtype=np.int64)
    nxt = 0
    for s in range(N):  # seeds in ascending cell order -> canonical numbering
        if lab[s] >= 0:
            continue
        lab[s] = nxt
        dq = collections.deque([s])
        while dq:
            c = dq.popleft()
            i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
            for di, dj, dk in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
                a, b, e = i + di, j + dj, k + dk
                if 0 <= a < nx and 0 <= b < ny and 0 <= e < nz:
                    n = a + nx * (b + ny * e)
                    if lab[n] < 0 and bins[n] == bins[c]:
                        lab[n] = nxt
                        dq.append(n)
        nxt += 1
    return lab, nxt


def test_indicator_brute_force_components():
    rng = np.random.default_rng(11)
    nx, ny, nz = 6, 5, 4
    ind = rng.uniform(-3, 3, nx * ny * nz)
    edges = [0.5, 2.0]
    part, M = opart.indicator_partition(ind, nx, ny, nz, edges, max_blocks=10 ** 6)
    a = np.abs(ind)
    bins = (a >= 0.5).astype(int) + (a >= 2.0)
    lab, n = _bfs_components(bins, nx, ny, nz)
    assert M == n and np.array_equal(part, lab)


def test_indicator_merge_respects_max_blocks():
    rng = np.random.default_rng(5)
    ind = rng.uniform(0, 2, 8 * 8 * 3)
    part, M = opart.indicator_partition(ind, 8, 8, 3, [1.0], max_blocks=8)
    assert M <= 8
    # every block is one bin
    bins = (np.abs(ind) >= 1.0).astype(int)
    for j in range(M):
        assert len(np.unique(bins[part == j])) == 1


def test_indicator_edges_must_increase():
    with pytest.raises(ValueError):
        opart.indicator_partition(np.zeros(4), 4, 1, 1, [2.0, 1.0])


# ---------------------------------------------------------------- dilated supports
def _chain_AT(T):
    """Flux matrix of a 1D chain with face transmissibilities T."""
    n = len(T) + 1
    A = sp.lil_matrix((n, n))
    for f, t in enumerate(T):
        A[f, f] += t
        A[f + 1, f + 1] += t
        A[f, f + 1] -= t
        A[f + 1, f] -= t
    return A.tocsr()


def test_dilation_spec_examples():
    """SPEC.md:424-426."""
    A = _chain_AT([1.0, 1.0, 1.0])
    part = np.array([0, 0, 1, 1])
    S0 = osup.dilated_pattern(part, 2, A, 0).toarray()
    assert np.array_equal(S0, np.array([[1, 0], [1, 0], [0, 1], [0, 1]]))
    S1 = osup.dilated_pattern(part, 2, A, 1).toarray()
    assert np.flatnonzero(S1[:, 0]).tolist() == [0, 1, 2]
    assert np.flatnonzero(S1[:, 1]).tolist() == [1, 2, 3]
    S9 = osup.dilated_pattern(part, 2, A, 9).toarray()
    assert S9.all()


def test_dilation_stops_at_sealing_face():
    A = _chain_AT([1.0, 0.0, 1.0])  # face (1, 2) sealed
    part = np.array([0, 0, 1, 1])
    S = osup.dilated_pattern(part, 2, A, 3).toarray()
    assert np.flatnonzero(S[:, 0]).tolist() == [0, 1]
    assert np.flatnonzero(S[:, 1]).tolist() == [2, 3]


def test_dilation_requirement_two_and_brute_force():
    p = random_problem(4, 7, 6, 4, (3, 3, 2), sigma=1.0)
    A_T, A, q, _ = tpfa.build(p)
    part, M = opart.wells_partition(p.nx, p.ny, p.nz, p.wells(), 1)
    for halo in (0, 1, 2):
        S = osup.dilated_pattern(part, M, A_T, halo)
        assert osup.check_requirements(part, S) == 0
        # brute force: graph distance <= halo from block j
        G = (A_T != 0).astype(int).tolil()
        adj = [set(G.rows[c]) - {c} for c in range(p.N)]
        for j in range(M):
            dist = {c: 0 for c in np.flatnonzero(part == j)}
            frontier = list(dist)
            for h in range(1, halo + 1):
                nf = []
                for c in frontier:
                    for n in adj[c]:
                        if n not in dist:
                            dist[n] = h
                            nf.append(n)
                frontier = nf
            assert sorted(dist) == np.flatnonzero(S[:, j].toarray().ravel()).tolist()


# ---------------------------------------------------------------- general MsRSB level
def test_general_single_block_is_ones():
    """single block -> P = column of ones, unchanged by smoothing."""
    p = random_problem(2, 6, 5, 3, (2, 2, 2))
    A_T, A, q, _ = tpfa.build(p)
    li = opl.general_level(p, A_T, np.zeros(p.N, dtype=np.int64), 1, 2, sweeps=10, fixed=True)
    assert np.all(li["P"].vals == 1.0)


def test_general_two_blocks_1d_partition_of_unity_and_symmetry():
    """homogeneous 1D, 2 blocks of 5 cells, full supports: P sums to one
    and decays monotonically across the overlap; by symmetry P_0(i) = P_1(9 - i)."""
    A = _chain_AT([1.0] * 9)

    class _P:  # minimal problem facts for general_level
        omega, sweep_tol, max_sweeps, fixed_sweeps = 2.0 / 3.0, 1e-8, 5000, False
    part = np.array([0] * 5 + [1] * 5)
    li = opl.general_level(_P, A, part, 2, 10, sweeps=5000, fixed=False)
    P = li["P"].dense()
    assert np.allclose(P.sum(axis=1), 1.0, atol=1e-14)
    assert np.all(np.diff(P[:, 0]) <= 1e-12)
    assert np.allclose(P[:, 0], P[::-1, 1], atol=1e-12)


def test_general_no_leak_across_barrier():
    """a sealing face bisecting a support -> no leak beyond it."""
    A = _chain_AT([1.0, 1.0, 1.0, 0.0, 1.0, 1.0, 1.0])

    class _P:
        omega, sweep_tol, max_sweeps, fixed_sweeps = 2.0 / 3.0, 1e-10, 500, False
    part = np.array([0, 0, 1, 1, 1, 1, 2, 2])
    li = opl.general_level(_P, A, part, 3, 3, sweeps=500, fixed=True)
    P = li["P"].dense()
    assert np.all(P[4:, 0] <= 1e-8) and np.all(P[:4, 2] <= 1e-8)


def test_static_levels_cut_iterations():
    """PAPER.md:373 / :437: static partitions honouring permeability contrasts and wells
    reduce the iteration count (small config-2 recipe)."""
    base = dict(shape=(12, 22, 20), max_sweeps=100, max_iter=20000)
    r0 = opl.run(make_problem(2, **base))
    W = {"kind": "wells", "radius": 2, "halo": 2}
    I = {"kind": "indicator", "edges": (1.0, 2.5), "halo": 0, "max_blocks": 256}
    r1 = opl.run(make_problem(2, static_levels=(W, I), **base))
    assert r0["sol"]["converged"] and r1["sol"]["converged"]
    assert r1["sol"]["iters"] < r0["sol"]["iters"]
