"""O5 — support regions S_j and the prolongation sparsity pattern.

Requirement 2: Ω_j ⊂ S_j ⊂ ∪ Ω_k.  The paper leaves the
construction to its MsRSB citation; readings:

A3 (Cartesian, BASELINE.json configs[0] "block plus neighbour blocks within the
box spanned by the neighbour block centres"): the OPEN box whose per-axis
limits are the neighbouring blocks' centres, extended to the domain boundary
where there is no neighbour.  In doubled integer coordinates (cell x has centre
2x+1; block J spanning cells [lo_J, hi_J) has centre C(J) = lo_J + hi_J):
    x ∈ S_J along axis a  ⇔  lo_a(J) < 2x+1 < hi_a(J),
    lo_a(J) = C(J-1) if J > 0 else -inf,   hi_a(J) = C(J+1) if J < n_a-1 else +inf.
Built here by the literal per-axis test and a tensor (Kronecker) product.

A4 (fault-split level): S_j = cells reachable from Ω_j inside the parent
Cartesian support box without crossing a face whose multiplier is not 1.

Patterns are returned as scipy CSR (N x M) boolean-valued matrices with sorted
column indices.  TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

from .grid import all_faces
from .partition import block_counts


def axis_membership(n, b):
    """Boolean (n x n_blocks) matrix: mem[x, J] = (lo(J) < 2x+1 < hi(J))."""
    nb = block_counts(n, b)
    lo_c = np.arange(nb) * b
    hi_c = np.minimum(lo_c + b, n)
    C = lo_c + hi_c                                  # doubled centres
    mem = np.zeros((n, nb), dtype=bool)
    for J in range(nb):
        lo = C[J - 1] if J > 0 else -np.inf
        hi = C[J + 1] if J < nb - 1 else np.inf
        for x in range(n):
            mem[x, J] = lo < 2 * x + 1 < hi
    return mem


def box_pattern(nx, ny, nz, block):
    """Open-box support pattern of the Cartesian partition (reading A3)."""
    mx = sp.csr_matrix(axis_membership(nx, block[0]).astype(np.int8))
    my = sp.csr_matrix(axis_membership(ny, block[1]).astype(np.int8))
    mz = sp.csr_matrix(axis_membership(nz, block[2]).astype(np.int8))
    S = sp.kron(mz, sp.kron(my, mx, format="csr"), format="csr")
    S.eliminate_zeros()
    S.sort_indices()
    S.data[:] = 1
    return S


def _pattern_from_pairs(rows, cols, N, M):
    S = sp.csr_matrix((np.ones(len(rows), dtype=np.int8), (rows, cols)), shape=(N, M))
    S.sum_duplicates()
    S.sort_indices()
    S.data[:] = 1
    return S


def flood_pattern(prob, parent_part, parent_pattern, split_part, Ms):
    """Support pattern of the fault-split level (reading A4)."""
    N = prob.N
    pp = parent_pattern.tocoo()
    node_cell = pp.row.astype(np.int64)
    node_par = pp.col.astype(np.int64)
    Mp = parent_pattern.shape[1]
    key = node_cell * Mp + node_par
    order = np.argsort(key)
    key_sorted = key[order]

    def node_of(cell, par):
        k = cell * Mp + par
        pos = np.searchsorted(key_sorted, k)
        pos = np.minimum(pos, len(key_sorted) - 1)
        ok = key_sorted[pos] == k
        return np.where(ok, order[pos], -1)

    # edges between (i, J) and (l, J) for non-fault faces with both ends in box J
    faces = all_faces(prob.nx, prob.ny, prob.nz)
    mults = (prob.mult_x, prob.mult_y, prob.mult_z)
    ea, eb = [], []
    indptr, indices = parent_pattern.indptr, parent_pattern.indices
    for a in range(3):
        left, right = faces[a]
        m = mults[a] if mults[a] is not None else np.ones(len(left))
        sel = m == 1.0
        left, right = left[sel], right[sel]
        cnt = indptr[left + 1] - indptr[left]
        rep_left = np.repeat(left, cnt)
        rep_right = np.repeat(right, cnt)
        starts = np.repeat(indptr[left], cnt)
        offs = np.arange(len(rep_left)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        par = indices[starts + offs].astype(np.int64)
        na = node_of(rep_left, par)
        nb = node_of(rep_right, par)
        ok = (na >= 0) & (nb >= 0)
        ea.append(na[ok])
        eb.append(nb[ok])
    ea, eb = np.concatenate(ea), np.concatenate(eb)
    nn = len(node_cell)
    g = sp.coo_matrix((np.ones(len(ea)), (ea, eb)), shape=(nn, nn))
    _, comp = connected_components(g, directed=False)

    # (component, child) pairs from the children's own cells
    cells = np.arange(N)
    own_nodes = node_of(cells, parent_part)
    assert np.all(own_nodes >= 0), "requirement 2 violated by parent pattern"
    pairs = np.unique(np.stack([comp[own_nodes], split_part]), axis=1)
    pc, pj = pairs[0], pairs[1]
    # every node inherits every child attached to its component
    n_comp = comp.max() + 1
    cnt = np.bincount(pc, minlength=n_comp)
    start = np.concatenate([[0], np.cumsum(cnt)])
    node_cnt = cnt[comp]
    rows = np.repeat(node_cell, node_cnt)
    base = np.repeat(start[comp], node_cnt)
    offs = np.arange(len(rows)) - np.repeat(np.cumsum(node_cnt) - node_cnt, node_cnt)
    cols = pj[base + offs]
    return _pattern_from_pairs(rows, cols, N, Ms)


def dilated_pattern(part, M, A_T, halo):
    """NEXT-3 supports of a general partition (requirement 2 of
    PAPER.md:220; reading B8): S_j = Ω_j dilated by `halo` layers of the graph of A_T
    (cells joined by a face with T != 0, so a sealing fault also bounds the support)."""
    N = len(part)
    part = np.asarray(part, dtype=np.int64)
    S = sp.csr_matrix((np.ones(N), (np.arange(N), part)), shape=(N, M))
    G = sp.csr_matrix(A_T, copy=True)
    G.eliminate_zeros()  # a face with T = 0 is no edge
    G.data[:] = 1.0
    G = (G + sp.identity(N, format="csr")).tocsr()
    for _ in range(halo):
        S = (G @ S).tocsr()
        S.data[:] = 1.0
    S.eliminate_zeros()
    S.sort_indices()
    return S.astype(np.int8)


def check_requirements(part, pattern):
    """Requirement 1–2 checks: every cell's own block column is
    in its row of the pattern.  Returns the number of violations."""
    N = len(part)
    own = pattern[np.arange(N), part]
    return int(N - np.count_nonzero(np.asarray(own).ravel()))
