"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct NumPy/SciPy (fp64, single thread) implementation
of what the MsRSB + iterative multiscale hot path computes, written from the
paper and the readings recorded in DESIGN.md §3 (SURVEY.md §8.c,
A1–A22).  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it.  The product package
`paper_2001_01624_b200` never imports it and shares no code with it; the two
meet only in the seeded input generator `synth/`.

Modules (step numbers follow SURVEY.md §8.c, O1–O12):
    grid       O1   natural ordering, faces per axis
    tpfa       O2-3 two-point transmissibilities, flux matrix A_T, gauge
    partition  O4   Cartesian, fault-split, Δp-binned (dynamic) partitions
    support    O5   open-box supports, flood-fill supports, CSR pattern
    basis      O6-7 restricted smoothing (MsRSB) sweeps
    coarse     O8   Galerkin A_c = P^T A P and its direct factorisation
    cycle      O9-11 multibasis Richardson iteration (Eq. 8) + dynamic stage
    transport  O12  config-4 sequential two-phase outer loop
    cost       Eq. (9) operation-count model

Parity pins: see tests/test_oracle_*.py.  Parity-unpinned functions are marked
"parity unpinned" in their docstrings and in DESIGN.md §3.4.
"""
import os as _os

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    _os.environ.setdefault(_v, "1")
