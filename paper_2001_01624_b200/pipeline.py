"""Whole-path driver over the C ABI for one synth.Problem (used by bench.py,
__graft_entry__.smoke and the GPU parity tests).  Setup order follows the paper:
build_tpfa -> partition/support -> smooth_basis -> coarse_assemble -> ms_iterate."""
from __future__ import annotations

import numpy as np

from .api import Context, Level, Operator, Solver


def problem_K(prob):
    return np.ascontiguousarray(np.concatenate([prob.kx, prob.ky, prob.kz]))


def problem_mult(prob):
    if prob.mult_x is None and prob.mult_y is None and prob.mult_z is None:
        return None
    nx, ny, nz = prob.nx, prob.ny, prob.nz
    mx = prob.mult_x if prob.mult_x is not None else np.ones((nx - 1) * ny * nz)
    my = prob.mult_y if prob.mult_y is not None else np.ones(nx * (ny - 1) * nz)
    mz = prob.mult_z if prob.mult_z is not None else np.ones(nx * ny * (nz - 1))
    return np.ascontiguousarray(np.concatenate([mx, my, mz]))


def build_operator(ctx: Context, prob, K=None, mult=None, mob=None):
    K = problem_K(prob) if K is None else K
    mult = problem_mult(prob) if mult is None else mult
    return Operator(ctx, prob.nx, prob.ny, prob.nz, K, prob.src_cells, prob.src_rates,
                    mult=mult, mob=mob, dx=prob.dx, dy=prob.dy, dz=prob.dz)


def build_levels(ctx: Context, op: Operator, prob, sweeps=None, fixed=None):
    """Cartesian level (+ fault-split level) smoothed and assembled."""
    ms = prob.max_sweeps if sweeps is None else sweeps
    fx = prob.fixed_sweeps if fixed is None else fixed
    tol = -1.0 if fx else prob.sweep_tol
    cart = Level.cartesian(ctx, op, prob.block)
    info = [cart.smooth(op, ms, prob.omega, tol)]
    levels = [cart]
    if prob.split_level:
        sp = Level.split(ctx, op, cart)
        # the split level starts from its own indicator (O6) and is smoothed the same way
        info.append(sp.smooth(op, ms, prob.omega, tol))
        levels.append(sp)
    for lv in levels:
        lv.assemble(op)
    return levels, info


def make_solver(ctx: Context, op: Operator, levels, prob):
    return Solver(ctx, op, levels, omega_s=prob.omega_s, nu=prob.nu,
                  post_smooth=prob.post_smooth, dynamic=prob.dynamic, edges=prob.dyn_edges,
                  max_blocks=prob.dyn_max_blocks)


def run(ctx: Context, prob, sweeps=None, fixed_sweeps=None, fixed_iters=None, max_iter=None,
        x0=None):
    """Full hot path; returns dict(op, levels, sweep_info, solver, x, sol)."""
    import torch

    op = build_operator(ctx, prob)
    levels, sweep_info = build_levels(ctx, op, prob, sweeps, fixed_sweeps)
    solver = make_solver(ctx, op, levels, prob)
    x = torch.zeros(prob.N, dtype=torch.float64, device=f"cuda:{ctx.device}")
    if x0 is not None:
        x.copy_(torch.as_tensor(x0))
    fi = prob.fixed_iters if fixed_iters is None else fixed_iters
    mi = prob.max_iter if max_iter is None else max_iter
    sol = solver.iterate(x, None, prob.cycle_tol, mi, fi)
    return dict(op=op, levels=levels, sweep_info=sweep_info, solver=solver, x=x, sol=sol)
