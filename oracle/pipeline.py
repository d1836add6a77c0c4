"""End-to-end oracle for one synth.Problem: O1–O11 in the paper's order.

build_tpfa -> Cartesian partition + open-box supports -> P^0 -> smoothing ->
(fault-split level) -> A_c per level -> multibasis Richardson (+ dynamic stage).
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import numpy as np

from . import basis as _basis
from . import partition as _part
from . import support as _sup
from . import tpfa as _tpfa
from .cycle import Level, iterate


def cartesian_level(prob, A_T, sweeps=None, fixed=None):
    part, M, _ = _part.cartesian(prob.nx, prob.ny, prob.nz, prob.block)
    pat = _sup.box_pattern(prob.nx, prob.ny, prob.nz, prob.block)
    P0 = _basis.indicator(part, pat)
    ms = prob.max_sweeps if sweeps is None else sweeps
    fx = prob.fixed_sweeps if fixed is None else fixed
    P, n, deltas = _basis.smooth(P0, A_T, prob.omega, ms, prob.sweep_tol, fx)
    return dict(part=part, M=M, pattern=pat, P=P, sweeps=n, deltas=deltas)


def split_level(prob, A_T, cart, sweeps=None, fixed=None):
    spart, Ms = _part.fault_split(prob, cart["part"])
    pat = _sup.flood_pattern(prob, cart["part"], cart["pattern"], spart, Ms)
    P0 = _basis.indicator(spart, pat)
    ms = prob.max_sweeps if sweeps is None else sweeps
    fx = prob.fixed_sweeps if fixed is None else fixed
    P, n, deltas = _basis.smooth(P0, A_T, prob.omega, ms, prob.sweep_tol, fx)
    return dict(part=spart, M=Ms, pattern=pat, P=P, sweeps=n, deltas=deltas)


def general_level(prob, A_T, part, M, halo, sweeps=None, fixed=None):
    """NEXT-3 level on a general partition: MsRSB from the constant basis on the
    dilated supports."""
    pat = _sup.dilated_pattern(part, M, A_T, halo)
    P0 = _basis.indicator(np.asarray(part, dtype=np.int64), pat)
    ms = prob.max_sweeps if sweeps is None else sweeps
    fx = prob.fixed_sweeps if fixed is None else fixed
    P, n, deltas = _basis.smooth(P0, A_T, prob.omega, ms, prob.sweep_tol, fx)
    return dict(part=np.asarray(part, dtype=np.int64), M=M, pattern=pat, P=P, sweeps=n,
                deltas=deltas)


def static_partition(prob, spec):
    """Partition of one NEXT-3 static level spec (synth.Problem.static_levels)."""
    if spec["kind"] == "wells":
        return _part.wells_partition(prob.nx, prob.ny, prob.nz, prob.wells(), spec["radius"])
    if spec["kind"] == "indicator":
        return _part.indicator_partition(prob.indicator(spec.get("field", "logk")), prob.nx,
                                         prob.ny, prob.nz, spec["edges"],
                                         spec.get("max_blocks", 1024))
    raise ValueError(f"unknown static level kind {spec['kind']!r}")


def run(prob, sweeps=None, fixed_sweeps=None, fixed_iters=None, max_iter=None,
        record_dynamic=False, x0=None, coarse="lu", assoc="right", levels_info=None,
        diag_order="assembly"):
    """coarse / assoc / diag_order: alternate exact coarse solver / A_c summation order /
    diagonal summation order of A (oracle.coarse, oracle.tpfa; floor measurement only).
    levels_info: reuse the smoothed levels of an earlier run (the alternates differ only
    after smoothing)."""
    A_T, A, q, trans = _tpfa.build(prob, diag_order=diag_order)
    if levels_info is not None:
        return _solve(prob, A_T, A, q, trans, levels_info, fixed_iters, max_iter,
                      record_dynamic, x0, coarse, assoc)
    cart = cartesian_level(prob, A_T, sweeps, fixed_sweeps)
    levels_info = [cart]
    if prob.split_level:
        levels_info.append(split_level(prob, A_T, cart, sweeps, fixed_sweeps))
    for spec in prob.static_levels:  # NEXT-3 (reading B11: after the general levels)
        part, M = static_partition(prob, spec)
        levels_info.append(general_level(prob, A_T, part, M, spec["halo"], sweeps, fixed_sweeps))
    return _solve(prob, A_T, A, q, trans, levels_info, fixed_iters, max_iter, record_dynamic,
                  x0, coarse, assoc)


def _solve(prob, A_T, A, q, trans, levels_info, fixed_iters, max_iter, record_dynamic, x0,
           coarse, assoc):
    levels = [Level(li["P"].matrix(), A, coarse, assoc) for li in levels_info]
    dyn = None
    if prob.dynamic:
        dyn = dict(nx=prob.nx, ny=prob.ny, nz=prob.nz, edges=prob.dyn_edges,
                   max_blocks=prob.dyn_max_blocks)
    fi = prob.fixed_iters if fixed_iters is None else fixed_iters
    mi = prob.max_iter if max_iter is None else max_iter
    x0 = np.zeros(prob.N) if x0 is None else x0
    smoother = make_smoother(prob, A)
    sol = iterate(A, q, x0, levels, prob.omega_s, prob.nu, prob.post_smooth,
                  prob.cycle_tol, mi, fi, dyn, record_dynamic, smoother, coarse, assoc)
    return dict(A_T=A_T, A=A, q=q, trans=trans, levels_info=levels_info, levels=levels,
                sol=sol, smoother=smoother)


def make_smoother(prob, A):
    """None = damped Jacobi (A9); "ilu0" = red-black ILU(0) (NEXT-2, reading B12)."""
    if prob.smoother == "jacobi":
        return None
    if prob.smoother == "ilu0":
        from .ilu import RBILU0
        return RBILU0(A, prob.nx, prob.ny, prob.nz)
    raise ValueError(f"unknown smoother {prob.smoother!r}")
