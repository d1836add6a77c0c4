"""O4 / O11 — coarse partitions.

* Cartesian ("general"): block index floor(x_a / b_a) per axis;
  ragged last block allowed (n_a need not divide).  Block id is natural order
  over the block grid.  Requirement 1: non-overlapping.
* Fault-split ("static"): connected components of each
  Cartesian block over faces whose multiplier is exactly 1 (reading A4/A20).
* Dynamic: cells binned by
  |Δp| against edges {0.1, 0.5}*max|Δp| (bin = number of edges <= |Δp_i|,
  reading A14), split into connected components over 6-neighbour (4 in 2D)
  adjacency between equal bins, small components merged per bin (reading A15).

Every numbering is canonical: ascending minimum cell index.
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

from .grid import all_faces


def block_counts(n, b):
    return -(-n // b)


def cartesian(nx, ny, nz, block):
    """Return (part[N] int64, M, (nbx, nby, nbz))."""
    bx, by, bz = block
    nbx, nby, nbz = block_counts(nx, bx), block_counts(ny, by), block_counts(nz, bz)
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    part = (i // bx) + nbx * ((j // by) + nby * (k // bz))
    return part.ravel().astype(np.int64), nbx * nby * nbz, (nbx, nby, nbz)


def canonical_relabel(labels):
    """Renumber arbitrary labels so that block ids ascend with each block's
    minimum cell index."""
    labels = np.asarray(labels)
    uniq, inv = np.unique(labels, return_inverse=True)
    mins = np.full(len(uniq), np.iinfo(np.int64).max)
    np.minimum.at(mins, inv, np.arange(len(labels)))
    order = np.argsort(mins, kind="stable")
    rank = np.empty(len(uniq), dtype=np.int64)
    rank[order] = np.arange(len(uniq))
    return rank[inv], len(uniq)


def _components(N, left, right, keep):
    g = sp.coo_matrix((np.ones(int(keep.sum())), (left[keep], right[keep])), shape=(N, N))
    _, lab = connected_components(g, directed=False)
    return lab


def fault_split(prob, part):
    """Components of each block over faces with multiplier == 1 (A4/A20)."""
    faces = all_faces(prob.nx, prob.ny, prob.nz)
    mults = (prob.mult_x, prob.mult_y, prob.mult_z)
    L, R, K = [], [], []
    for a in range(3):
        left, right = faces[a]
        m = mults[a] if mults[a] is not None else np.ones(len(left))
        L.append(left)
        R.append(right)
        K.append((m == 1.0) & (part[left] == part[right]))
    left, right, keep = np.concatenate(L), np.concatenate(R), np.concatenate(K)
    lab = _components(prob.N, left, right, keep)
    return canonical_relabel(lab)


def dp_bins(dp, edges=(0.1, 0.5)):
    """bin_i = #{e in edges*max|dp| : e <= |dp_i|} (A14); edges as fp64 products."""
    a = np.abs(dp)
    m = a.max() if len(a) else 0.0
    b = np.zeros(len(a), dtype=np.int64)
    for e in edges:
        b += (a >= e * m)
    return b, m


def dynamic_partition(dp, nx, ny, nz, edges=(0.1, 0.5), max_blocks=1024):
    """Δp-binned constant-basis partition (A14, A15).

    Returns (part, M_dyn) or (None, 0) when max|dp| == 0 (stage skipped)."""
    bins, m = dp_bins(dp, edges)
    if m == 0.0:
        return None, 0
    return _bin_components(bins, nx, ny, nz, max_blocks)


def indicator_partition(ind, nx, ny, nz, edges, max_blocks=1024):
    """NEXT-3 static partition from a per-cell indicator ("agglomerates
    cells into coarse blocks based on a flow indicator"): bin_i =
    #{e in edges : e <= |ind_i|} with ABSOLUTE edges (reading B10), then the same
    components and small-component rule as the dynamic partition (A15)."""
    edges = list(edges)
    if any(b <= a for a, b in zip(edges, edges[1:])):
        raise ValueError("edges must be strictly increasing")
    a = np.abs(np.asarray(ind, dtype=np.float64))
    bins = np.zeros(len(a), dtype=np.int64)
    for e in edges:
        bins += (a >= e)
    return _bin_components(bins, nx, ny, nz, max_blocks)


def wells_partition(nx, ny, nz, wells, radius):
    """NEXT-3 well partition ("one for each well plus one to ensure
    partition of unity"; reading B9): block w holds the cells whose
    Chebyshev index distance to the nearest perforation of well w is <= radius; a cell
    in reach of several wells joins the nearest, ties to the lower well index; block
    n_w holds every other cell and is omitted when empty.  Returns (part, M)."""
    if radius < 0:
        raise ValueError("radius must be >= 0")
    N = nx * ny * nz
    c = np.arange(N)
    i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
    best = np.full(N, np.iinfo(np.int64).max)
    owner = np.full(N, -1, dtype=np.int64)
    for w, cells in enumerate(wells):
        cells = np.asarray(cells, dtype=np.int64)
        if len(cells) == 0 or cells.min() < 0 or cells.max() >= N:
            raise ValueError("well outside the grid or without perforations")
        d = np.full(N, np.iinfo(np.int64).max)
        for q in cells:
            qi, qj, qk = q % nx, (q // nx) % ny, q // (nx * ny)
            d = np.minimum(d, np.maximum(np.maximum(np.abs(i - qi), np.abs(j - qj)), np.abs(k - qk)))
        take = d < best  # strict: an equal distance keeps the lower well index
        best[take] = d[take]
        owner[take] = w
    n_w = len(wells)
    part = np.where(best <= radius, owner, n_w)
    M = n_w + int(np.any(part == n_w))
    return part, M


def _bin_components(bins, nx, ny, nz, max_blocks):
    """Connected components of equal-bin cells over the grid faces, components smaller
    than s_min merged into one block per bin, s_min doubling from 1 until at most
    max_blocks blocks remain (A15); canonical numbering."""
    N = nx * ny * nz
    faces = all_faces(nx, ny, nz)
    left = np.concatenate([f[0] for f in faces])
    right = np.concatenate([f[1] for f in faces])
    keep = bins[left] == bins[right]
    lab = _components(N, left, right, keep)
    sizes = np.bincount(lab)
    s_min = 1
    while True:
        small = sizes[lab] < s_min
        # merged label per bin for small components: a value past all comp labels
        merged = np.where(small, len(sizes) + bins, lab)
        n_blocks = len(np.unique(merged))
        if n_blocks <= max_blocks or s_min > N:
            break
        s_min *= 2
    return canonical_relabel(merged)
