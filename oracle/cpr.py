"""NEXT-4 — CPR two-stage preconditioner for compressible two-phase flow (oracle).

Follows, in the paper's order:
  * the discrete equations, PAPER.md:87-100 (§3, Eq. residual-equations and
    accumulation): F_β^i = A_β^i + Σ_j G_β^{i,j} − Q_β^i with
    A_β^i = (φ ρ_β S_β)_i^{n+1} − (φ ρ_β S_β)_i^n,
    G_β^{i,j} = (Δt/|Ω_i|) |Γ_ij| (ρ_β v_β·n)_ij,  Q_β^i = (Δt/|Ω_i|) q_β^i,
    two-point fluxes with single-point upstream mobility;
  * the Newton system and its block form, PAPER.md:111-137 (Eq. fim-system);
  * IMPES / quasi-IMPES weights and the premultiplication by W, PAPER.md:163-202 (§4);
  * the two-stage solution procedure, PAPER.md:287-292 (decoupling, predictor = one or a
    few cycles of the iterative multiscale multibasis method on J*_pp, corrector = a
    smoother on the full system), with the operations of SPEC.md:293-354 (cpr module).

Model readings (C1-C6): two phases w, o with one component each
(X_αβ = δ_αβ), no gravity, no capillary pressure; unknowns x = (p_1..p_N, S_1..S_N),
S = S_w, S_o = 1 − S; ρ_α(p) = ρ_α^0 exp(c_α (p − p_ref)), φ(p) = φ^0 exp(c_r (p − p_ref));
λ_w = S^n/μ_w, λ_o = (1 − S)^n/μ_o with n = 2 (the config-4 curves) or 1; upstream cell of face (l, r) is l
when p_l ≥ p_r (ties to the left cell, reading A17); wells: an injector cell (rate Q > 0)
injects water, q_w = ρ_w(p_i) Q, q_o = 0; a producer (Q < 0) produces at its own
fractional flow, q_α = ρ_α(p_i) f_α(S_i) Q with f_α = λ_α/(λ_w + λ_o).  Equation order
F = (F_w, F_o): the first block row is the one premultiplied (the pressure equation).

The Jacobian is the complex-step derivative of this residual (Squire & Trapp: the
imaginary part of F(x + i h e_k) / h is ∂F/∂x_k to rounding, no cancellation), with a
27-colouring of the cells so that one evaluation yields many columns.  It shares nothing
with the device path's analytic derivatives.
TEST INFRASTRUCTURE ONLY.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular

from .cycle import stage
from .ilu import ilu0, rb_permutation


@dataclasses.dataclass
class Fluid:
    """Fluid and rock constants of the compressible two-phase model (reading C1)."""
    mu_w: float = 1.0
    mu_o: float = 5.0
    rho_w: float = 1000.0      # ρ_w^0 at p_ref
    rho_o: float = 800.0       # ρ_o^0 at p_ref
    c_w: float = 4e-5          # 1/pressure unit
    c_o: float = 1e-4
    c_r: float = 3e-5
    phi: float = 0.2           # φ^0 at p_ref
    p_ref: float = 100.0
    dt: float = 0.05           # Δt
    nrel: int = 2              # relative-permeability exponent: k_rw = S^n, k_ro = (1-S)^n


# ----------------------------------------------------------------------------- properties


def density(fl, p, phase):
    rho0, c = (fl.rho_w, fl.c_w) if phase == 0 else (fl.rho_o, fl.c_o)
    return rho0 * np.exp(c * (p - fl.p_ref))


def porosity(fl, p):
    return fl.phi * np.exp(fl.c_r * (p - fl.p_ref))


def mobility(fl, S, phase):
    """λ_w = S^n/μ_w, λ_o = (1 − S)^n/μ_o, n = 2 (the config-4 curves) or 1 (linear)."""
    if fl.nrel not in (1, 2):
        raise ValueError("nrel must be 1 or 2")
    s = S if phase == 0 else 1.0 - S
    kr = s * s if fl.nrel == 2 else s
    return kr / (fl.mu_w if phase == 0 else fl.mu_o)


# ----------------------------------------------------------------------------- residual


def accumulation(fl, p, S, p_n, S_n):
    """A_β^i = (φ ρ_β S_β)^{n+1} − (φ ρ_β S_β)^n for β = w, o."""
    phi, phi_n = porosity(fl, p), porosity(fl, p_n)
    Aw = phi * density(fl, p, 0) * S - phi_n * density(fl, p_n, 0) * S_n
    Ao = phi * density(fl, p, 1) * (1.0 - S) - phi_n * density(fl, p_n, 1) * (1.0 - S_n)
    return Aw, Ao


def residual(fl, prob, trans, p, S, p_n, S_n, well_cells, well_rates):
    """(F_w, F_o), each of length N; complex inputs give complex outputs (complex step).

    trans: oracle.tpfa.transmissibilities(prob) (T_f = |Γ| K-harmonic, no mobility)."""
    vol = prob.dx * prob.dy * prob.dz
    s = fl.dt / vol
    Aw, Ao = accumulation(fl, p, S, p_n, S_n)
    Fw = np.array(Aw, dtype=np.result_type(Aw, np.float64), copy=True)
    Fo = np.array(Ao, dtype=Fw.dtype, copy=True)
    for left, right, T in trans:
        if len(left) == 0:
            continue
        dp = p[left] - p[right]
        up_left = np.real(p[left]) >= np.real(p[right])  # ties to the left cell (A17)
        up = np.where(up_left, left, right)
        for Fb, ph in ((Fw, 0), (Fo, 1)):
            m = density(fl, p[up], ph) * mobility(fl, S[up], ph)
            flux = s * T * m * dp            # G_β^{l,r}: from l towards r
            np.add.at(Fb, left, flux)
            np.add.at(Fb, right, -flux)
    # sources: Q_β^i = (Δt/|Ω_i|) q_β^i
    for c, Q in zip(np.asarray(well_cells).tolist(), np.asarray(well_rates).tolist()):
        if Q > 0:
            Fw[c] -= s * density(fl, p[c], 0) * Q
        elif Q < 0:
            lw, lo = mobility(fl, S[c], 0), mobility(fl, S[c], 1)
            Fw[c] -= s * density(fl, p[c], 0) * (lw / (lw + lo)) * Q
            Fo[c] -= s * density(fl, p[c], 1) * (lo / (lw + lo)) * Q
    return Fw, Fo


# ----------------------------------------------------------------------------- Jacobian


def _colour(nx, ny, nz):
    c = np.arange(nx * ny * nz)
    i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
    return (i % 3) + 3 * (j % 3) + 9 * (k % 3)


def _neighbours(nx, ny, nz):
    """nb[d, c] for d = centre, -x, +x, -y, +y, -z, +z (or -1)."""
    N = nx * ny * nz
    c = np.arange(N)
    i, j, k = c % nx, (c // nx) % ny, c // (nx * ny)
    nb = np.full((7, N), -1, dtype=np.int64)
    nb[0] = c
    nb[1] = np.where(i > 0, c - 1, -1)
    nb[2] = np.where(i < nx - 1, c + 1, -1)
    nb[3] = np.where(j > 0, c - nx, -1)
    nb[4] = np.where(j < ny - 1, c + nx, -1)
    nb[5] = np.where(k > 0, c - nx * ny, -1)
    nb[6] = np.where(k < nz - 1, c + nx * ny, -1)
    return nb


def jacobian(fl, prob, trans, p, S, p_n, S_n, well_cells, well_rates, h=1e-30):
    """J = ∂(F_w, F_o)/∂(p, S) as a 2N x 2N CSR matrix, rows (F_w | F_o), columns (p | S),
    every 7-point stencil entry of all four blocks stored (explicit zeros kept)."""
    nx, ny, nz = prob.nx, prob.ny, prob.nz
    N = nx * ny * nz
    col = _colour(nx, ny, nz)
    nb = _neighbours(nx, ny, nz)
    vals = np.zeros((2, 2, 7, N))  # [row block β, column block v, stencil d, row cell]
    for cc in range(27):
        sel = col == cc
        if not sel.any():
            continue
        for v in range(2):
            pz = p.astype(np.complex128)
            Sz = S.astype(np.complex128)
            (pz if v == 0 else Sz)[sel] += 1j * h
            Fw, Fo = residual(fl, prob, trans, pz, Sz, p_n, S_n, well_cells, well_rates)
            for d in range(7):
                j = nb[d]
                ok = (j >= 0)
                ok[ok] = sel[j[ok]]
                vals[0, v, d, ok] = Fw.imag[ok] / h
                vals[1, v, d, ok] = Fo.imag[ok] / h
    rows, cols, data = [], [], []
    for b in range(2):
        for v in range(2):
            for d in range(7):
                ok = nb[d] >= 0
                rows.append(b * N + np.nonzero(ok)[0])
                cols.append(v * N + nb[d][ok])
                data.append(vals[b, v, d, ok])
    J = sp.coo_matrix((np.concatenate(data), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(2 * N, 2 * N)).tocsr()
    J.sort_indices()
    return J


def accumulation_saturation_derivative(fl, p, S, p_n, S_n, h=1e-30):
    """(∂A_w/∂S_i, ∂A_o/∂S_i) per cell (the accumulation is cell-local: one complex step)."""
    Aw, Ao = accumulation(fl, p.astype(np.complex128), S + 1j * h, p_n, S_n)
    return Aw.imag / h, Ao.imag / h


# ----------------------------------------------------------------------------- CPR (§4)


def weights(m1, m2):
    """Per cell, solve [m_{2,1} m_{2,2}; 1 1] [w_1; w_2] = [0; 1] (
    SPEC.md:306-315); a cell whose first row is identically zero gets w = (1, 0)."""
    m1 = np.asarray(m1, dtype=np.float64)
    m2 = np.asarray(m2, dtype=np.float64)
    w = np.zeros((2, len(m1)))
    for i in range(len(m1)):
        if m1[i] == 0.0 and m2[i] == 0.0:
            w[:, i] = (1.0, 0.0)
            continue
        Mi = np.array([[m1[i], m2[i]], [1.0, 1.0]])
        if np.linalg.det(Mi) == 0.0:
            raise ZeroDivisionError(f"singular CPR weight system in cell {i}")
        w[:, i] = np.linalg.solve(Mi, np.array([0.0, 1.0]))
    return w


def impes_weights(fl, p, S, p_n, S_n):
    """IMPES: Σ_β W_β ∂A_β/∂x_s = 0."""
    mw, mo = accumulation_saturation_derivative(fl, p, S, p_n, S_n)
    return weights(mw, mo)


def quasi_impes_weights(J, N):
    """quasi-IMPES: Σ_β W_β diag(∂F_β/∂x_s) = 0."""
    J = sp.csr_matrix(J)
    d = np.arange(N)
    mw = np.asarray(J[d, N + d]).ravel()
    mo = np.asarray(J[N + d, N + d]).ravel()
    return weights(mw, mo)


def premultiply(J, F, w):
    """J* = W J, F* = W F with W = [[W_1, W_2], [0, I]].

    Row i of the first block row is w_1,i J_w(i, :) + w_2,i J_o(i, :), formed entry by entry
    on J's block 7-point pattern so that entries which cancel to 0 (quasi-IMPES's diagonal
    coupling) stay in the pattern (reading C4: ILU(0)'s pattern is the block stencil)."""
    J = sp.csr_matrix(J)
    J.sort_indices()
    N = w.shape[1]
    n = 2 * N
    ip, ix, dv = J.indptr, J.indices, J.data
    rows = np.repeat(np.arange(n), np.diff(ip))
    if not np.array_equal(np.diff(ip[:N + 1]), np.diff(ip[N:])):
        raise ValueError("the two block rows of J do not share a pattern")
    a0, a1 = ip[0], ip[N]
    if not np.array_equal(ix[a0:a1], ix[a1:]):
        raise ValueError("the two block rows of J do not share a pattern")
    r0 = rows[a0:a1]
    top = w[0][r0] * dv[a0:a1] + w[1][r0] * dv[a1:]
    Js = sp.csr_matrix((np.concatenate([top, dv[a1:]]), ix.copy(), ip.copy()), shape=(n, n))
    F = np.asarray(F, dtype=np.float64)
    Fs = np.concatenate([w[0] * F[:N] + w[1] * F[N:], F[N:]])
    return Js, Fs


def block_rb_ilu0(Js, nx, ny, nz):
    """ILU(0) of the full system J* (2N x 2N) with the two unknowns of a cell adjacent and
    the cells in red-black order (reading B12 extended to the coupled system, C4): the
    textbook IKJ elimination (oracle.ilu.ilu0) of the permuted matrix.  Returns (L, U, q)
    with q[new] = old unknown index."""
    N = nx * ny * nz
    rb = rb_permutation(nx, ny, nz)
    q = np.empty(2 * N, dtype=np.int64)
    q[0::2] = rb          # p of the m-th cell in red-black order
    q[1::2] = N + rb      # S of that cell
    Jp = sp.csr_matrix(Js)[q][:, q]
    L, U = ilu0(Jp)
    return L, U, q


class CPR:
    """The two-stage preconditioner.

    levels: oracle.cycle.Level objects built on J*_pp (R = P^T, A_c = P^T J*_pp P);
    apply(r): predictor Δx_p = n_cycles Eq.-(8) cycles from zero on J*_pp Δx_p = r_p,
    residual update r' = r − J*[:, :N] Δx_p, corrector Δx = (Δx_p, 0) + (LU)^{-1} r'."""

    def __init__(self, Js, N, levels, nx, ny, nz, n_cycles=1, omega_s=2.0 / 3.0, nu=1,
                 pressure_solve=None, corrector=None):
        self.Js = sp.csr_matrix(Js)
        self.N = N
        self.Jpp = self.Js[:N, :N].tocsr()
        self.Jcol_p = self.Js[:, :N].tocsr()
        self.DA = self.Jpp.diagonal()
        self.levels = levels
        self.n_cycles = n_cycles
        self.omega_s = omega_s
        self.nu = nu
        self.pressure_solve = pressure_solve   # optional exact pressure solver (pins)
        if corrector is None:
            L, U, q = block_rb_ilu0(self.Js, nx, ny, nz)
            self.L, self.U, self.q = L, U, q
            corrector = self._ilu_solve
        self.corrector = corrector

    def _ilu_solve(self, r):
        rp = np.asarray(r, dtype=np.float64)[self.q]
        y = spsolve_triangular(self.L, rp, lower=True)
        e = spsolve_triangular(self.U, y, lower=False)
        out = np.empty_like(e)
        out[self.q] = e
        return out

    def predictor(self, rp):
        if self.pressure_solve is not None:
            return self.pressure_solve(rp)
        z = np.zeros_like(rp)
        for _ in range(self.n_cycles):
            for lev in self.levels:
                z = stage(self.Jpp, self.DA, rp, z, lev, self.omega_s, self.nu, False)
        return z

    def apply(self, r):
        r = np.asarray(r, dtype=np.float64)
        dxp = self.predictor(r[:self.N])
        r2 = r - self.Jcol_p @ dxp
        dx = self.corrector(r2)
        dx[:self.N] += dxp
        return dx
