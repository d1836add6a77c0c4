"""Config recipes (BASELINE.json configs[0..4]).

Every field is float64, natural cell order c = i + nx*(j + ny*k),
z index 0 is the top layer.  Face arrays follow the per-axis face order
    x-faces: f = i + (nx-1)*(j + ny*k)   joins cells (i,j,k) and (i+1,j,k)
    y-faces: f = i + nx*(j + (ny-1)*k)   joins (i,j,k) and (i,j+1,k)
    z-faces: f = i + nx*(j + ny*k)       joins (i,j,k) and (i,j,k+1)
The recipes draw random numbers only; no transmissibility, basis or solver
arithmetic lives here.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np


@dataclasses.dataclass
class Problem:
    name: str
    nx: int
    ny: int
    nz: int
    kx: np.ndarray
    ky: np.ndarray
    kz: np.ndarray
    src_cells: np.ndarray          # int64, cell indices
    src_rates: np.ndarray          # float64, + injection / - production (per cell)
    block: tuple                   # coarse block size (bx, by, bz)
    dx: float = 1.0
    dy: float = 1.0
    dz: float = 1.0
    phi: float = 0.2
    mult_x: Optional[np.ndarray] = None   # per x-face multipliers (None = all ones)
    mult_y: Optional[np.ndarray] = None
    mult_z: Optional[np.ndarray] = None
    # method parameters of the config (BASELINE.json configs)
    omega: float = 2.0 / 3.0
    max_sweeps: int = 300
    sweep_tol: float = 1e-3
    fixed_sweeps: bool = False            # config 1: exactly max_sweeps sweeps
    omega_s: float = 2.0 / 3.0
    nu: int = 1
    post_smooth: bool = False
    split_level: bool = False             # config 3: fault-split second stage
    dynamic: bool = False                 # config 3: dynamic Δp stage
    cycle_tol: float = 1e-6
    max_iter: int = 5000
    fixed_iters: int = 0                  # config 5: exactly 20 iterations
    dyn_edges: tuple = (0.1, 0.5)
    dyn_max_blocks: int = 1024
    # NEXT-3 static levels after the general ones, e.g. ({"kind": "wells", "radius": 2,
    # "halo": 2}, {"kind": "indicator", "edges": (1.0,), "halo": 1, "max_blocks": 512})
    static_levels: tuple = ()
    smoother: str = "jacobi"              # "jacobi" (A9) or "ilu0" (NEXT-2, the paper's)

    @property
    def N(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def n_faces(self) -> int:
        nx, ny, nz = self.nx, self.ny, self.nz
        return (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)

    def wells(self):
        """Perforated cells grouped into wells: one well per (i, j) column of source
        cells (fully penetrating 5-spot columns; a 2D source cell is its own well),
        in order of first appearance."""
        cols = {}
        for c in self.src_cells.tolist():
            key = c % (self.nx * self.ny)
            cols.setdefault(key, []).append(c)
        return [np.array(v, dtype=np.int64) for v in cols.values()]

    def indicator(self, field="logk"):
        """Per-cell static indicator: "logk" = log10(kx / min kx) >= 0 (the permeability
        flow indicator of PAPER.md:360)."""
        if field != "logk":
            raise ValueError(field)
        return np.log10(self.kx / self.kx.min())

    def rhs(self) -> np.ndarray:
        q = np.zeros(self.N)
        np.add.at(q, self.src_cells, self.src_rates)
        return q


# ----------------------------------------------------------------------------- helpers


def _box3_truncated(g: np.ndarray) -> np.ndarray:
    """3x3 (2D) box mean over in-grid neighbours (truncated window)."""
    s = np.zeros_like(g)
    c = np.zeros_like(g)
    ny, nx = g.shape
    for dj in (-1, 0, 1):
        for di in (-1, 0, 1):
            ys = slice(max(0, dj), ny + min(0, dj))
            yd = slice(max(0, -dj), ny + min(0, -dj))
            xs = slice(max(0, di), nx + min(0, di))
            xd = slice(max(0, -di), nx + min(0, -di))
            s[yd, xd] += g[ys, xs]
            c[yd, xd] += 1.0
    return s / c


def _standardise(g: np.ndarray) -> np.ndarray:
    return (g - g.mean()) / g.std()


def _gauss_smooth(noise: np.ndarray, std: float) -> np.ndarray:
    from scipy.ndimage import gaussian_filter

    return gaussian_filter(noise, sigma=std, mode="reflect")


def _five_spot(nx: int, ny: int, nz: int, rate_inj: float = 4.0, rate_prod: float = -1.0):
    """Fully penetrating 5-spot columns: injector at (nx//2, ny//2),
    producers at the four corner columns.  Sum of rates is exactly zero."""
    cols = [((nx // 2, ny // 2), rate_inj),
            ((0, 0), rate_prod), ((nx - 1, 0), rate_prod),
            ((0, ny - 1), rate_prod), ((nx - 1, ny - 1), rate_prod)]
    cells, rates = [], []
    for (i, j), r in cols:
        for k in range(nz):
            cells.append(i + nx * (j + ny * k))
            rates.append(r)
    return np.asarray(cells, dtype=np.int64), np.asarray(rates, dtype=np.float64)


def _channels(rng, nx: int, ny: int, nz_chan: int, frac: float = 0.30) -> np.ndarray:
    """Binary sinuous-channel facies, ribbons along y."""
    mask = np.zeros((nz_chan, ny, nx), dtype=bool)
    ys = np.arange(ny)[:, None]
    xs = np.arange(nx)[None, :] + 0.5
    guard = 0
    while mask.mean() < frac and guard < 10000:
        guard += 1
        x0 = rng.uniform(0, nx)
        a = rng.uniform(2, 10)
        lam = rng.uniform(40, 120)
        ph = rng.uniform(0, 2 * np.pi)
        w = rng.uniform(3, 8)
        t = int(rng.integers(2, 7))
        t = min(t, nz_chan)
        top = int(rng.integers(0, nz_chan - t + 1))
        centre = x0 + a * np.sin(2 * np.pi * ys / lam + ph)
        plane = np.abs(xs - centre) <= 0.5 * w
        mask[top:top + t] |= plane[None, :, :]
    return mask


# ----------------------------------------------------------------------------- recipes


def _config1(shape=None, seed=1, **kw) -> Problem:
    nx, ny = shape[:2] if shape else (64, 64)
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((ny, nx))
    g = _standardise(_box3_truncated(g))
    k = np.exp(g).ravel()
    cells = np.array([0, nx * ny - 1], dtype=np.int64)
    rates = np.array([1.0, -1.0])
    p = Problem(name="config1", nx=nx, ny=ny, nz=1, kx=k.copy(), ky=k.copy(), kz=k.copy(),
                src_cells=cells, src_rates=rates, block=(8, 8, 1),
                max_sweeps=200, fixed_sweeps=True, sweep_tol=0.0)
    return _override(p, kw)


def _perm_config2(rng, nx, ny, nz):
    nz_top = min(35, nz) if nz == 85 else max(1, (nz * 35) // 85)
    nz_bot = nz - nz_top
    noise = rng.standard_normal((nz_top, ny, nx))
    g = _standardise(_gauss_smooth(noise, 5.0))
    k = np.empty((nz, ny, nx))
    k[:nz_top] = np.exp(1.5 * g)
    if nz_bot > 0:
        ch = _channels(rng, nx, ny, nz_bot)
        k[nz_top:] = np.where(ch, 1000.0, 1.0)
    return k.ravel()


def _config2(shape=None, seed=2, **kw) -> Problem:
    nx, ny, nz = shape if shape else (60, 220, 85)
    rng = np.random.default_rng(seed)
    k = _perm_config2(rng, nx, ny, nz)
    cells, rates = _five_spot(nx, ny, nz)
    p = Problem(name="config2", nx=nx, ny=ny, nz=nz, kx=k.copy(), ky=k.copy(), kz=k.copy(),
                src_cells=cells, src_rates=rates, block=(6, 11, 5))
    return _override(p, kw)


def fault_multipliers(nx, ny, nz, faults):
    """faults: list of (axis, plane_index, lo, hi, value).  axis 'x': plane between
    i=plane and i+1 for lo <= j < hi; axis 'y': plane between j=plane and j+1 for
    lo <= i < hi.  All z."""
    mx = np.ones((nz, ny, nx - 1))
    my = np.ones((nz, ny - 1, nx))
    for axis, plane, lo, hi, val in faults:
        if axis == "x":
            mx[:, lo:hi, plane] = val
        else:
            my[:, plane, lo:hi] = val
    return mx.ravel(), my.ravel(), np.ones(nx * ny * max(nz - 1, 0))


def _config3(shape=None, seed=2, **kw) -> Problem:
    p = _config2(shape, seed)
    nx, ny, nz = p.nx, p.ny, p.nz
    if (nx, ny, nz) == (60, 220, 85):
        faults = [("x", 19, 0, 154, 0.0), ("x", 39, 66, 220, 0.0),
                  ("y", 72, 0, 60, 1e-3), ("y", 146, 0, 60, 1e-3)]
    else:
        # proportional placement on reduced grids; partial planes end on block
        # boundaries (multiples of by) as in the full config
        by = p.block[1]
        # planes placed strictly inside coarse blocks so that they split them
        fx1, fx2 = nx // 3, min(nx - 2, (2 * nx) // 3 + 1)
        nby = -(-ny // by)
        j1 = by * max(1, (7 * nby) // 10)
        j2 = by * max(1, (3 * nby) // 10)
        fy1, fy2 = ny // 3, min(ny - 2, (2 * ny) // 3 + 1)
        faults = [("x", fx1, 0, min(j1, ny), 0.0), ("x", fx2, min(j2, ny), ny, 0.0),
                  ("y", fy1, 0, nx, 1e-3), ("y", fy2, 0, nx, 1e-3)]
    mx, my, mz = fault_multipliers(nx, ny, nz, faults)
    p.name = "config3"
    p.mult_x, p.mult_y, p.mult_z = mx, my, mz
    p.post_smooth = True
    p.split_level = True
    p.dynamic = True
    return _override(p, kw)


def _config4(shape=None, seed=2, **kw) -> Problem:
    p = _config2(shape, seed)
    p.name = "config4"
    return _override(p, kw)


def _config5(shape=None, seed=5, **kw) -> Problem:
    nx, ny, nz = shape if shape else (200, 400, 125)
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal((nz, ny, nx))
    g = _standardise(_gauss_smooth(noise, 5.0))
    del noise
    kx = np.exp(2.0 * g).ravel()
    del g
    a = rng.uniform(0.01, 0.1, size=nx * ny * nz)
    kz = kx * a
    cells, rates = _five_spot(nx, ny, nz)
    p = Problem(name="config5", nx=nx, ny=ny, nz=nz, kx=kx, ky=kx.copy(), kz=kz,
                src_cells=cells, src_rates=rates, block=(10, 10, 5), fixed_iters=20)
    return _override(p, kw)


def _override(p: Problem, kw) -> Problem:
    for k, v in kw.items():
        if not hasattr(p, k):
            raise AttributeError(k)
        setattr(p, k, v)
    return p


CONFIGS = {1: _config1, 2: _config2, 3: _config3, 4: _config4, 5: _config5}


def make_problem(config: int, shape=None, seed=None, **overrides) -> Problem:
    """Build config `config` (1..5) at its BASELINE.json size, or at a reduced `shape`
    with the same recipe (parity tests)."""
    f = CONFIGS[config]
    kwargs = {} if seed is None else {"seed": seed}
    return f(shape, **kwargs, **overrides)


def random_problem(seed: int, nx: int, ny: int, nz: int, block, sigma: float = 1.0,
                   faults=None, **overrides) -> Problem:
    """Small fuzz problem: iid log-normal K, 5-spot (3D) or corner pair (2D)."""
    rng = np.random.default_rng(seed)
    n = nx * ny * nz
    kx = np.exp(sigma * rng.standard_normal(n))
    ky = np.exp(sigma * rng.standard_normal(n))
    kz = np.exp(sigma * rng.standard_normal(n))
    if nz == 1 or nx * ny < 9:
        cells = np.array([0, n - 1], dtype=np.int64)
        rates = np.array([1.0, -1.0])
    else:
        cells, rates = _five_spot(nx, ny, nz)
    p = Problem(name=f"random{seed}", nx=nx, ny=ny, nz=nz, kx=kx, ky=ky, kz=kz,
                src_cells=cells, src_rates=rates, block=tuple(block))
    if faults:
        p.mult_x, p.mult_y, p.mult_z = fault_multipliers(nx, ny, nz, faults)
    return _override(p, overrides)


# ----------------------------------------------------------------------------- NEXT-4 state


@dataclasses.dataclass
class CprState:
    """A synthetic Newton state of the compressible two-phase model (NEXT-4): current
    iterate (p, S), previous time level (p_n, S_n), well cells and volumetric rates."""
    p: np.ndarray
    S: np.ndarray
    p_n: np.ndarray
    S_n: np.ndarray
    well_cells: np.ndarray
    well_rates: np.ndarray


def cpr_state(prob: Problem, seed: int = 11, p_ref: float = 100.0, dp: float = 20.0,
              rate: float = 2.0) -> CprState:
    """Seeded smooth random pressure (p_ref ± dp) and saturation (0.05..0.95) fields on the
    problem's grid, a previous time level a small random step away, and the problem's
    5-spot cells with rates scaled by `rate`.  Random numbers only."""
    rng = np.random.default_rng(seed)
    shape = (prob.nz, prob.ny, prob.nx)
    sig = max(1.0, min(prob.nx, prob.ny) / 8.0)

    def field():
        g = _gauss_smooth(rng.standard_normal(shape), sig)
        return _standardise(g).ravel() if g.std() > 0 else g.ravel()

    p = p_ref + dp * np.tanh(field() / 2.0)
    S = 0.05 + 0.9 / (1.0 + np.exp(-field()))
    p_n = p - 0.5 * np.abs(field())
    S_n = np.clip(S - 0.05 * rng.uniform(0.0, 1.0, size=S.size), 0.0, 1.0)
    return CprState(p=p, S=S, p_n=p_n, S_n=S_n, well_cells=prob.src_cells.copy(),
                    well_rates=rate * prob.src_rates)
