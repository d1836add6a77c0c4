"""Oracle pins — partitions and supports (O4, O5, O11 partition).

Requirements 1–2; SPEC.md:383-391, :407-409 examples;
open-box support rule (reading A3) on hand-worked 1D cases; fault-split and
dynamic partitions against an independent pure-Python BFS on tiny grids."""
import json
import os
from collections import deque

import numpy as np
import pytest

from oracle import partition, support
from synth.configs import make_problem, random_problem

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_cartesian_counts_and_ragged():
    part, M, nb = partition.cartesian(42, 22, 1, (7, 11, 1))   # PAPER.md:300 6x2 partition
    assert M == 12 and nb == (6, 2, 1)
    part, M, nb = partition.cartesian(23, 17, 7, (5, 4, 3))
    assert nb == (5, 5, 3) and M == 75
    assert part[22 + 23 * (16 + 17 * 6)] == 74
    assert np.bincount(part, minlength=M).min() > 0              # every block nonempty


def test_open_box_membership_hand():
    # n=10, b=5: doubled centres C(0)=5, C(1)=15 → S_0: 2x+1 < 15 (x<=6); S_1: 2x+1 > 5 (x>=3)
    m = support.axis_membership(10, 5)
    assert list(np.nonzero(m[:, 0])[0]) == list(range(0, 7))
    assert list(np.nonzero(m[:, 1])[0]) == list(range(3, 10))
    # n=8, b=4 (even): C(0)=4, C(1)=12 → S_0 = {0..5}, S_1 = {2..7}
    m = support.axis_membership(8, 4)
    assert list(np.nonzero(m[:, 0])[0]) == list(range(0, 6))
    assert list(np.nonzero(m[:, 1])[0]) == list(range(2, 8))
    # ragged: n=7, b=3 → blocks [0,3),[3,6),[6,7); C = 3, 9, 13
    m = support.axis_membership(7, 3)
    assert list(np.nonzero(m[:, 0])[0]) == [0, 1, 2, 3]          # 2x+1 < 9
    assert list(np.nonzero(m[:, 1])[0]) == [2, 3, 4, 5]          # 3 < 2x+1 < 13
    assert list(np.nonzero(m[:, 2])[0]) == [5, 6]                # 2x+1 > 9


def test_config_pattern_sizes():
    """nnz(P) and M of configs 1 and 2 (SURVEY.md §8.a sizes table)."""
    for cfg, nnz, M, maxs in [(1, 14400, 64, 4), (2, 6964260, 3400, 8)]:
        p = make_problem(cfg) if cfg == 1 else None
        dims = (64, 64, 1, (8, 8, 1)) if cfg == 1 else (60, 220, 85, (6, 11, 5))
        S = support.box_pattern(*dims)
        assert S.nnz == nnz and S.shape[1] == M
        assert np.diff(S.indptr).max() == maxs


@pytest.mark.parametrize("dims", [(23, 17, 7, (5, 4, 3)), (30, 12, 1, (6, 4, 1))])
def test_requirement2_and_slots(dims):
    nx, ny, nz, blk = dims
    part, M, _ = partition.cartesian(nx, ny, nz, blk)
    S = support.box_pattern(nx, ny, nz, blk)
    assert support.check_requirements(part, S) == 0
    dim = sum(n > 1 for n in (nx, ny, nz))
    assert np.diff(S.indptr).max() <= 2 ** dim


def _bfs_labels(N, adj_ok):
    """Independent brute-force BFS component labelling, numbered by min cell."""
    lab = -np.ones(N, dtype=np.int64)
    nxt = 0
    for s in range(N):
        if lab[s] >= 0:
            continue
        lab[s] = nxt
        dq = deque([s])
        while dq:
            c = dq.popleft()
            for l in adj_ok(c):
                if lab[l] < 0:
                    lab[l] = nxt
                    dq.append(l)
        nxt += 1
    return lab, nxt


def _nbrs(c, nx, ny, nz):
    i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
    out = []
    if i > 0: out.append(c - 1)
    if i < nx - 1: out.append(c + 1)
    if j > 0: out.append(c - nx)
    if j < ny - 1: out.append(c + nx)
    if k > 0: out.append(c - nx * ny)
    if k < nz - 1: out.append(c + nx * ny)
    return out


def test_fault_split_vs_bfs():
    faults = [("x", 1, 0, 6, 0.0), ("y", 2, 0, 12, 1e-3), ("x", 9, 2, 10, 0.0)]
    p = random_problem(7, 12, 10, 3, (4, 5, 3), faults=faults)
    part, M, _ = partition.cartesian(p.nx, p.ny, p.nz, p.block)
    sp_, Ms = partition.fault_split(p, part)
    nx, ny, nz = p.nx, p.ny, p.nz
    mx = p.mult_x.reshape(nz, ny, nx - 1)
    my = p.mult_y.reshape(nz, ny - 1, nx)

    def ok(c):
        i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
        out = []
        for l in _nbrs(c, nx, ny, nz):
            li, lj = l % nx, (l // nx) % ny
            if li != i:
                m = mx[k, j, min(i, li)]
            elif lj != j:
                m = my[k, min(j, lj), i]
            else:
                m = 1.0
            if m == 1.0 and part[l] == part[c]:
                out.append(l)
        return out

    lab, n = _bfs_labels(p.N, ok)
    assert Ms == n and Ms > M
    assert np.array_equal(sp_, lab)


def test_dynamic_spec_examples():
    g = json.load(open(os.path.join(GOLD, "dynamic_spec_examples.json")))
    for case in g["cases"]:
        dp = np.array(case["dp"])
        part, M = partition.dynamic_partition(dp, len(dp), 1, 1)
        assert M == case["n_blocks"]
        assert list(part) == case["part"]


def test_dynamic_zero_dp_skips():
    part, M = partition.dynamic_partition(np.zeros(10), 10, 1, 1)
    assert part is None and M == 0


def test_dynamic_vs_bfs_and_merge():
    rng = np.random.default_rng(3)
    nx, ny, nz = 9, 7, 4
    dp = rng.standard_normal(nx * ny * nz) ** 3
    part, M = partition.dynamic_partition(dp, nx, ny, nz)
    bins, _ = partition.dp_bins(dp)
    lab, n = _bfs_labels(nx * ny * nz,
                         lambda c: [l for l in _nbrs(c, nx, ny, nz) if bins[l] == bins[c]])
    assert M == n and np.array_equal(part, lab)
    # merge rule (A15): cap the count → small comps merged into one block per bin
    part2, M2 = partition.dynamic_partition(dp, nx, ny, nz, max_blocks=5)
    assert M2 <= 5
    for blk in range(M2):
        assert len(np.unique(bins[part2 == blk])) == 1               # one bin per block
    first = np.array([np.min(np.nonzero(part2 == b)[0]) for b in range(M2)])
    assert np.all(np.diff(first) > 0)                                # canonical numbering


def test_split_pattern_requirements():
    p = make_problem(3, shape=(18, 22, 10))
    part, M, _ = partition.cartesian(p.nx, p.ny, p.nz, p.block)
    S = support.box_pattern(p.nx, p.ny, p.nz, p.block)
    sp_, Ms = partition.fault_split(p, part)
    F = support.flood_pattern(p, part, S, sp_, Ms)
    assert support.check_requirements(sp_, F) == 0
    # support of a split block stays inside its parent's box
    parent_of = np.zeros(Ms, dtype=np.int64)
    parent_of[sp_] = part
    Fc = F.tocoo()
    Sd = S.tocsr()
    inside = np.asarray(Sd[Fc.row, parent_of[Fc.col]]).ravel()
    assert np.all(inside == 1)


def test_flood_pattern_vs_bfs():
    """A4 by brute force: S_j = cells reachable from Ω_j inside the parent box
    without crossing a face whose multiplier != 1."""
    faults = [("x", 1, 0, 6, 0.0), ("y", 2, 0, 12, 1e-3), ("x", 5, 3, 10, 0.0)]
    p = random_problem(11, 12, 10, 2, (4, 5, 2), faults=faults)
    nx, ny, nz = p.nx, p.ny, p.nz
    part, M, _ = partition.cartesian(nx, ny, nz, p.block)
    S = support.box_pattern(nx, ny, nz, p.block).toarray() > 0
    sp_, Ms = partition.fault_split(p, part)
    F = support.flood_pattern(p, part, support.box_pattern(nx, ny, nz, p.block), sp_, Ms)
    F = F.toarray() > 0
    mx = p.mult_x.reshape(nz, ny, nx - 1)
    my = p.mult_y.reshape(nz, ny - 1, nx)

    def face_ok(c, l):
        i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
        li, lj = l % nx, (l // nx) % ny
        if li != i:
            return mx[k, j, min(i, li)] == 1.0
        if lj != j:
            return my[k, min(j, lj), i] == 1.0
        return True

    for j in range(Ms):
        J = part[np.nonzero(sp_ == j)[0][0]]
        seen = set(np.nonzero(sp_ == j)[0].tolist())
        dq = deque(seen)
        while dq:
            c = dq.popleft()
            for l in _nbrs(c, nx, ny, nz):
                if l not in seen and S[l, J] and face_ok(c, l):
                    seen.add(l)
                    dq.append(l)
        assert set(np.nonzero(F[:, j])[0].tolist()) == seen
