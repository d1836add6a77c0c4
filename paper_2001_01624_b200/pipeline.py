"""Whole-path driver over the C ABI for one synth.Problem (used by bench.py,
__graft_entry__.smoke and the GPU parity tests).  Setup order follows the paper:
build_tpfa -> partition/support -> smooth_basis -> coarse_assemble -> ms_iterate."""
from __future__ import annotations

import numpy as np

from .api import Context, Level, Operator, Solver, partition_indicator, partition_wells


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
    for spec in prob.static_levels:  # NEXT-3, after the general levels (reading B11)
        part, M = static_partition(ctx, op, prob, spec)
        lv = Level.general(ctx, op, part, M, spec["halo"])
        info.append(lv.smooth(op, ms, prob.omega, tol))
        levels.append(lv)
    for lv in levels:
        lv.assemble(op)
    return levels, info


def static_partition(ctx: Context, op: Operator, prob, spec):
    """Partition of one NEXT-3 static level spec on the GPU; inputs (well perforations,
    the indicator field) come from the problem definition (synth)."""
    if spec["kind"] == "wells":
        return partition_wells(ctx, prob.nx, prob.ny, prob.nz, prob.wells(), spec["radius"])
    if spec["kind"] == "indicator":
        ind = np.ascontiguousarray(prob.indicator(spec.get("field", "logk")), dtype=np.float64)
        return partition_indicator(ctx, op, ind, spec["edges"], spec.get("max_blocks", 1024))
    raise ValueError(f"unknown static level kind {spec['kind']!r}")


def make_solver(ctx: Context, op: Operator, levels, prob):
    return Solver(ctx, op, levels, omega_s=prob.omega_s, nu=prob.nu,
                  post_smooth=prob.post_smooth, dynamic=prob.dynamic, edges=prob.dyn_edges,
                  max_blocks=prob.dyn_max_blocks, smoother=prob.smoother)


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


def run_sequential(ctx: Context, prob, steps=100, k_adapt=5, mu_w=1.0, mu_o=5.0,
                   pv_per_step=0.005, init_sweeps=None, init_fixed=None, fixed_iters=None,
                   max_iter=None, keep_states=False):
    """Config 4 (row a12): per step, face mobility -> k_adapt warm sweeps of the reused
    basis on A_T(λ) -> RAP + factor -> ms_iterate from the previous
    pressure -> explicit upwind transport -> upstream mobility for the next step.
    fixed_iters: per-step iteration counts (lockstep parity mode) or None."""
    import torch

    dev = f"cuda:{ctx.device}"
    N = prob.N
    phi = torch.full((N,), float(prob.phi), dtype=torch.float64, device=dev)
    # the initial basis is config 2's (λ = 1); a uniform λ scales A_T and leaves the
    # smoothing update unchanged, so smoothing before or after the first λ is equivalent
    op = build_operator(ctx, prob)
    dt = op.step_size(phi, pv_per_step)
    # step 1: S = 0 everywhere, λ_t(0) = 1/μ_o on every face (reading A17)
    mob = op.upstream_mobility(None, None, mu_w, mu_o,
                               torch.empty(prob.n_faces, dtype=torch.float64, device=dev))
    cart = Level.cartesian(ctx, op, prob.block)
    ms = prob.max_sweeps if init_sweeps is None else init_sweeps
    fx = prob.fixed_sweeps if init_fixed is None else init_fixed
    n0 = cart.smooth(op, ms, prob.omega, -1.0 if fx else prob.sweep_tol)[0]
    op.set_mobility(mob)
    S = torch.zeros(N, dtype=torch.float64, device=dev)
    x = torch.zeros(N, dtype=torch.float64, device=dev)
    mi = prob.max_iter if max_iter is None else max_iter
    recs = []
    for n in range(steps):
        cart.smooth(op, k_adapt, prob.omega, -1.0)
        cart.assemble(op)
        solver = Solver(ctx, op, [cart], omega_s=prob.omega_s, nu=prob.nu,
                        post_smooth=prob.post_smooth)
        fi = int(fixed_iters[n]) if fixed_iters is not None else 0
        sol = solver.iterate(x, None, prob.cycle_tol, mi, fi, history=False)
        solver.close()
        nsub = op.transport_upwind(x, S, phi, mu_w, mu_o, dt, mob_out=mob)
        op.set_mobility(mob)
        rec = dict(iters=sol["iters"], status=sol["status"], n_sub=nsub)
        if keep_states:
            rec.update(p=x.cpu().numpy(), S=S.cpu().numpy(), mob=mob.cpu().numpy())
        recs.append(rec)
    return dict(steps=recs, dt=dt, init_sweeps=n0, op=op, level=cart, x=x, S=S)
