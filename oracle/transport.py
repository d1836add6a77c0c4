"""O12 — config 4: sequential incompressible two-phase outer loop.

PAPER.md:39-41 (sequential splitting: a pressure step, then transport at fixed
total velocity), PAPER.md:101 ("single-point upstream evaluation for the interface
mobilities"), PAPER.md:277 (the basis is reused and adapted by "iterating a few
times extra"); BASELINE.json configs[3] (λ = S²/μ_w + (1-S)²/μ_o, μ_w = 1, μ_o = 5,
explicit upwind saturation between 100 pressure steps).  Readings:

A17  face mobility λ_f = λ_t(S_up), upstream by the sign of the previous step's face
     flux (ties, F = 0, take the left/lower cell); step 1 uses S = 0 everywhere.
     A_T(λ) = Σ_f T_f λ_f (e_i - e_l)(e_i - e_l)^T stays symmetric.
A18  each step injects 0.005 pore volumes: dt = 0.005 PV / Σ q⁺.  Explicit upwind
     sub-steps h = dt / n_sub, n_sub = max(1, ceil(dt / dt_cfl)),
     dt_cfl = 0.5 min_i φ_i|Ω_i| / out_i,  out_i = Σ_faces max(F_out, 0) + max(-q_i, 0),
     divided by fw'_max = the largest forward-difference slope of f_w on S = k/1000.
     Per sub-step:  S_i += h/(φ_i|Ω_i|) (Σ_in F f_w(S_up) - Σ_out F f_w(S_i)
                                        + q_i⁺ - q_i⁻ f_w(S_i)),
     the injector delivers pure water (f_w = 1).  k_adapt = 5 warm sweeps per step.

All plain NumPy loops over the three face arrays, fp64.  TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import math

import numpy as np

from . import basis as _basis
from . import tpfa as _tpfa
from .cycle import Level, iterate
from .grid import all_faces
from .pipeline import cartesian_level


def total_mobility(S, mu_w, mu_o):
    """λ_t = S²/μ_w + (1-S)²/μ_o (BASELINE.json configs[3])."""
    return S * S / mu_w + (1.0 - S) * (1.0 - S) / mu_o


def fractional_flow(S, mu_w, mu_o):
    """f_w = λ_w / λ_t."""
    lw = S * S / mu_w
    lo = (1.0 - S) * (1.0 - S) / mu_o
    return lw / (lw + lo)


def fw_slope_max(mu_w, mu_o, n=1000):
    """Largest forward-difference slope of f_w on the grid S = k/n (reading A18)."""
    s = np.arange(n + 1) / n
    f = fractional_flow(s, mu_w, mu_o)
    return float(np.max((f[1:] - f[:-1]) * n))


def face_fluxes(trans, p):
    """F_f = T_f (p_left - p_right) for every face; positive leaves the left cell."""
    return [(left, right, T * (p[left] - p[right])) for left, right, T in trans]


def cfl_substeps(fluxes, q, phi, vol, dt, mu_w, mu_o):
    out = np.maximum(-q, 0.0)
    for left, right, F in fluxes:
        np.add.at(out, left, np.maximum(F, 0.0))
        np.add.at(out, right, np.maximum(-F, 0.0))
    pos = out > 0.0
    if not np.any(pos):
        return 1
    m = float(np.min(phi[pos] * vol / out[pos]))
    dt_cfl = 0.5 * m / fw_slope_max(mu_w, mu_o)
    return max(1, int(math.ceil(dt / dt_cfl)))


def transport(trans, p, S, phi, q, vol, mu_w, mu_o, dt):
    """Explicit single-point-upstream water transport over dt (reading A18).

    Returns (S_new, n_sub)."""
    fluxes = face_fluxes(trans, p)
    n_sub = cfl_substeps(fluxes, q, phi, vol, dt, mu_w, mu_o)
    h = dt / n_sub
    S = np.array(S, dtype=np.float64, copy=True)
    for _ in range(n_sub):
        fS = fractional_flow(S, mu_w, mu_o)
        net = np.zeros_like(S)
        for left, right, F in fluxes:
            up = np.where(F > 0.0, left, right)
            water = F * fS[up]                 # water volume rate left -> right
            np.add.at(net, left, -water)
            np.add.at(net, right, water)
        net += np.where(q > 0.0, q, q * fS)    # injector: f_w = 1; producers: f_w(S_i)
        S = S + h / (phi * vol) * net
    return S, n_sub


def upstream_mobility(faces, p, S, mu_w, mu_o):
    """Per-face λ_t of the upstream cell (ties to the left cell), reading A17."""
    out = []
    for left, right in faces:
        up = np.where(p[left] - p[right] >= 0.0, left, right)
        out.append(total_mobility(S[up], mu_w, mu_o))
    return out


def step_size(prob, q, phi, pv_per_step=0.005):
    vol = prob.dx * prob.dy * prob.dz
    pv = float(np.sum(phi)) * vol
    return pv_per_step * pv / float(np.sum(q[q > 0.0]))


def run(prob, steps=100, k_adapt=5, mu_w=1.0, mu_o=5.0, pv_per_step=0.005,
        init_sweeps=None, init_fixed=None, fixed_iters=None, max_iter=None, coarse="lu"):
    """Config-4 outer loop.  fixed_iters: None, or a per-step list of iteration counts
    (lockstep mode, SURVEY.md §8.c protocol 5).  coarse: alternate exact coarse solver
    (oracle.coarse; floor measurement only).  Returns per-step records."""
    N = prob.N
    vol = prob.dx * prob.dy * prob.dz
    phi = np.full(N, prob.phi)
    q = prob.rhs()
    dt = step_size(prob, q, phi, pv_per_step)
    faces = all_faces(prob.nx, prob.ny, prob.nz)
    A_T0, _, _, _ = _tpfa.build(prob)
    cart = cartesian_level(prob, A_T0, init_sweeps, init_fixed)
    P = cart["P"]
    mob = [np.full(len(f[0]), total_mobility(0.0, mu_w, mu_o)) for f in faces]
    S = np.zeros(N)
    x = np.zeros(N)
    mi = prob.max_iter if max_iter is None else max_iter
    recs = []
    for n in range(steps):
        A_T, A, _, trans = _tpfa.build(prob, mob)
        P, _, _ = _basis.smooth(P, A_T, prob.omega, k_adapt, 0.0, fixed=True)
        lev = Level(P.matrix(), A, coarse)
        fi = fixed_iters[n] if fixed_iters is not None else 0
        sol = iterate(A, q, x, [lev], prob.omega_s, prob.nu, prob.post_smooth,
                      prob.cycle_tol, mi, fi)
        x = sol["x"]
        S, n_sub = transport(trans, x, S, phi, q, vol, mu_w, mu_o, dt)
        mob = upstream_mobility(faces, x, S, mu_w, mu_o)
        recs.append(dict(iters=sol["iters"], converged=sol["converged"], res=sol["res"][-1],
                         p=x.copy(), S=S.copy(), n_sub=n_sub,
                         mob=np.concatenate(mob)))
    return dict(steps=recs, dt=dt, init_sweeps=cart["sweeps"], P=P)
