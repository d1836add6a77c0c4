"""O1 — structured grid, natural ordering, faces per axis.

Follows SPEC.md:136-139 (natural ordering i + nx*j + nx*ny*k) and
SPEC.md:150-158 (interior faces of the 6-point stencil; 3x3 grid has 12 faces,
2x1 has 1, 1x1 has 0).  TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np


def cell_index(i, j, k, nx, ny):
    return i + nx * (j + ny * k)


def cell_coords(c, nx, ny):
    c = np.asarray(c)
    return c % nx, (c // nx) % ny, c // (nx * ny)


def axis_faces(nx: int, ny: int, nz: int, axis: int):
    """Interior faces normal to `axis` (0=x, 1=y, 2=z) as (left_cell, right_cell)
    arrays, in the per-axis face order of synth/configs.py (left cell runs in
    natural order over the (n_a - 1)-shortened axis)."""
    shape = [nx, ny, nz]
    shape[axis] -= 1
    if shape[axis] <= 0:
        e = np.zeros(0, dtype=np.int64)
        return e, e
    k, j, i = np.meshgrid(np.arange(shape[2]), np.arange(shape[1]), np.arange(shape[0]),
                          indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    left = cell_index(i, j, k, nx, ny).astype(np.int64)
    off = (1, nx, nx * ny)[axis]
    return left, left + off


def all_faces(nx: int, ny: int, nz: int):
    """List of three (left, right) pairs, one per axis."""
    return [axis_faces(nx, ny, nz, a) for a in range(3)]
