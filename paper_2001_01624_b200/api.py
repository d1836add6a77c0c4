"""Thin Python binding over libmsb's C ABI (include/msb.h): argument marshalling
only.  Every arithmetic step of the hot path runs in the library's CUDA kernels.

Arrays may be torch tensors (CUDA or CPU) or NumPy arrays; they are passed to the
library as raw pointers (host or device — the library detects which).  Device
memory for the library's own handles comes from the PyTorch caching allocator
through the context's allocator hook.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

OK, NOT_CONVERGED = 0, 1
_ERRNAMES = {-1: "EINVAL", -2: "EDIM", -3: "EZERO_DIAG", -4: "ESINGULAR",
             -5: "EINCONSISTENT", -6: "EDIVERGED", -7: "ENOMEM", -8: "ECUDA"}


class MsbError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_ERRNAMES.get(code, code)}: {msg}")
        self.code = code


def _torch():
    import torch
    return torch


def _ptr(a, dtype=np.float64):
    """Raw pointer of a contiguous torch tensor / numpy array (None -> NULL)."""
    if a is None:
        return None
    torch = None
    try:
        import torch as _t
        torch = _t
    except Exception:  # pragma: no cover
        pass
    if torch is not None and isinstance(a, torch.Tensor):
        want = {np.float64: torch.float64, np.int32: torch.int32}[dtype]
        if a.dtype != want or not a.is_contiguous():
            raise TypeError(f"expected contiguous {want} tensor, got {a.dtype}")
        return C.c_void_p(a.data_ptr())
    if not isinstance(a, np.ndarray) or a.dtype != dtype or not a.flags.c_contiguous:
        raise TypeError(f"expected contiguous numpy {np.dtype(dtype)} array")
    return C.c_void_p(a.ctypes.data)


class Context:
    """msb_ctx on one CUDA device and stream (default: torch's current stream)."""

    def __init__(self, device: int = 0, stream=None, torch_alloc: bool = True):
        self.lib = L.load()
        torch = _torch()
        if not torch.cuda.is_available():
            raise MsbError(-8, "no CUDA device: libmsb has no CPU path")
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        handle = C.c_void_p(stream.cuda_stream)
        self._keep = []
        if torch_alloc:
            dev = device

            t_alloc = torch.cuda.caching_allocator_alloc
            t_free = torch.cuda.caching_allocator_delete
            stream_ = self.stream

            def _alloc(nbytes, user):
                try:
                    return t_alloc(int(nbytes), dev, stream_)
                except Exception:
                    return None

            def _free(ptr, user):
                try:
                    t_free(ptr)
                except Exception:  # interpreter shutdown: the process is exiting anyway
                    pass

            af, ff = L.ALLOC_FN(_alloc), L.FREE_FN(_free)
        else:
            af, ff = L.ALLOC_FN(), L.FREE_FN()
        self._keep += [af, ff]
        h = C.c_void_p()
        st = self.lib.msb_ctx_create(C.byref(h), device, handle, af, ff, None)
        if st != OK:
            raise MsbError(st, "msb_ctx_create failed")
        self.h = h

    def check(self, st: int, what: str) -> int:
        if st < 0:
            raise MsbError(st, f"{what}: {self.lib.msb_last_error(self.h).decode()}")
        return st

    def launch_count(self) -> int:
        return int(self.lib.msb_launch_count())

    def close(self):
        if getattr(self, "h", None):
            self.lib.msb_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _grid(nx, ny, nz, dx=1.0, dy=1.0, dz=1.0):
    return L.Grid(int(nx), int(ny), int(nz), float(dx), float(dy), float(dz))


class Operator:
    """build_tpfa(grid, K, wells) — row a1.  K: (3N,) float64 SoA kx|ky|kz."""

    def __init__(self, ctx: Context, nx, ny, nz, K, src_cells, src_rates, mult=None, mob=None,
                 dx=1.0, dy=1.0, dz=1.0):
        self.ctx = ctx
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.N = self.nx * self.ny * self.nz
        self.grid = _grid(nx, ny, nz, dx, dy, dz)
        cells = np.asarray(src_cells, dtype=np.int64)
        rates = np.asarray(src_rates, dtype=np.float64)
        arr = (L.Source * max(1, len(cells)))()
        for t, (c, r) in enumerate(zip(cells, rates)):
            arr[t].cell = int(c)
            arr[t].rate = float(r)
        h = C.c_void_p()
        st = ctx.lib.msb_build_tpfa(ctx.h, C.byref(self.grid), _ptr(K), _ptr(mult), _ptr(mob),
                                    arr, len(cells), C.byref(h))
        ctx.check(st, "msb_build_tpfa")
        self.h = h

    @property
    def n_faces(self):
        nx, ny, nz = self.nx, self.ny, self.nz
        return (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)

    def set_mobility(self, mob):
        self.ctx.check(self.ctx.lib.msb_op_set_mobility(self.ctx.h, self.h, _ptr(mob)),
                       "msb_op_set_mobility")

    def export(self):
        T = np.empty(self.n_faces)
        q = np.empty(self.N)
        self.ctx.check(self.ctx.lib.msb_op_export(self.ctx.h, self.h, _ptr(T), _ptr(q)),
                       "msb_op_export")
        return T, q

    def apply(self, x, y):
        self.ctx.check(self.ctx.lib.msb_op_apply(self.ctx.h, self.h, _ptr(x), _ptr(y)),
                       "msb_op_apply")

    def transport_upwind(self, p, S, phi, mu_w, mu_o, dt, mob_out=None):
        n = C.c_int32()
        self.ctx.check(self.ctx.lib.msb_transport_upwind(self.ctx.h, self.h, _ptr(p), _ptr(S),
                                                         _ptr(phi), float(mu_w), float(mu_o),
                                                         float(dt), _ptr(mob_out), C.byref(n)),
                       "msb_transport_upwind")
        return n.value

    def upstream_mobility(self, p, S, mu_w, mu_o, mob_out):
        """Per-face upstream λ_t (msb_upstream_mobility); p / S None = zero vectors."""
        self.ctx.check(self.ctx.lib.msb_upstream_mobility(self.ctx.h, self.h, _ptr(p), _ptr(S),
                                                          float(mu_w), float(mu_o),
                                                          _ptr(mob_out)),
                       "msb_upstream_mobility")
        return mob_out

    def step_size(self, phi, pv_per_step):
        """Config-4 step length dt (msb_transport_step_size)."""
        dt = C.c_double()
        self.ctx.check(self.ctx.lib.msb_transport_step_size(self.ctx.h, self.h, _ptr(phi),
                                                            float(pv_per_step), C.byref(dt)),
                       "msb_transport_step_size")
        return dt.value

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.msb_op_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partition_cartesian(ctx: Context, nx, ny, nz, block, part_out=None):
    g = _grid(nx, ny, nz)
    M = C.c_int32()
    ctx.check(ctx.lib.msb_partition_cartesian(ctx.h, C.byref(g), int(block[0]), int(block[1]),
                                              int(block[2]), _ptr(part_out, np.int32), C.byref(M)),
              "msb_partition_cartesian")
    return M.value


def partition_wells(ctx: Context, nx, ny, nz, wells, radius, part_out=None):
    """NEXT-3 well partition (msb_partition_wells); wells: sequence of cell-index arrays.
    Returns (part int32[N], M)."""
    g = _grid(nx, ny, nz)
    ptr = np.zeros(len(wells) + 1, dtype=np.int32)
    ptr[1:] = np.cumsum([len(w) for w in wells])
    cells = np.ascontiguousarray(np.concatenate([np.asarray(w) for w in wells]), dtype=np.int32)
    part = np.empty(nx * ny * nz, dtype=np.int32) if part_out is None else part_out
    M = C.c_int32()
    ctx.check(ctx.lib.msb_partition_wells(ctx.h, C.byref(g), _ptr(ptr, np.int32),
                                          _ptr(cells, np.int32), len(wells), int(radius),
                                          _ptr(part, np.int32), C.byref(M)), "msb_partition_wells")
    return part, M.value


def partition_indicator(ctx: Context, op: "Operator", ind, edges, max_blocks=1024, part_out=None):
    """NEXT-3 indicator partition (msb_partition_indicator).  Returns (part int32[N], M)."""
    e = np.ascontiguousarray(edges, dtype=np.float64)
    part = np.empty(op.N, dtype=np.int32) if part_out is None else part_out
    M = C.c_int32()
    ctx.check(ctx.lib.msb_partition_indicator(ctx.h, op.h, _ptr(ind), _ptr(e) if len(e) else None,
                                              len(e), int(max_blocks), _ptr(part, np.int32),
                                              C.byref(M)), "msb_partition_indicator")
    return part, M.value


class Level:
    """A (P, R = P^T, A_c) triple on one coarse partition."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.h = handle

    # --- constructors (row a2)
    @classmethod
    def cartesian(cls, ctx: Context, op: Operator, block):
        h = C.c_void_p()
        nnz = C.c_int64()
        ctx.check(ctx.lib.msb_level_create_cartesian(ctx.h, op.h, int(block[0]), int(block[1]),
                                                     int(block[2]), C.byref(h), C.byref(nnz)),
                  "msb_level_create_cartesian")
        lev = cls(ctx, h)
        lev.N = op.N
        return lev

    @classmethod
    def split(cls, ctx: Context, op: Operator, parent: "Level"):
        h = C.c_void_p()
        nnz = C.c_int64()
        ctx.check(ctx.lib.msb_level_create_split(ctx.h, op.h, parent.h, C.byref(h), C.byref(nnz)),
                  "msb_level_create_split")
        lev = cls(ctx, h)
        lev.N = op.N
        return lev

    @classmethod
    def constant(cls, ctx: Context, op: Operator, part, M: int):
        h = C.c_void_p()
        ctx.check(ctx.lib.msb_level_create_constant(ctx.h, op.h, _ptr(part, np.int32), int(M),
                                                    C.byref(h)), "msb_level_create_constant")
        lev = cls(ctx, h)
        lev.N = op.N
        return lev

    @classmethod
    def general(cls, ctx: Context, op: Operator, part, M: int, halo: int):
        """NEXT-3 level on a general partition: supports = blocks dilated by `halo` layers."""
        h = C.c_void_p()
        nnz = C.c_int64()
        ctx.check(ctx.lib.msb_level_create_general(ctx.h, op.h, _ptr(part, np.int32), int(M),
                                                   int(halo), C.byref(h), C.byref(nnz)),
                  "msb_level_create_general")
        lev = cls(ctx, h)
        lev.N = op.N
        return lev

    def info(self, with_part=False):
        M, nnz, W = C.c_int32(), C.c_int64(), C.c_int32()
        part = np.empty(self.N, dtype=np.int32) if with_part else None
        self.ctx.check(self.ctx.lib.msb_level_info(self.ctx.h, self.h, C.byref(M), C.byref(nnz),
                                                   C.byref(W), _ptr(part, np.int32)),
                       "msb_level_info")
        out = dict(M=M.value, nnz=nnz.value, W=W.value)
        if with_part:
            out["part"] = part
        return out

    # --- row a3
    def smooth(self, op: Operator, max_sweeps: int, omega: float = 2.0 / 3.0, tol: float = 1e-3):
        n = C.c_int32()
        last = C.c_double()
        deltas = np.zeros(max(1, max_sweeps))
        st = self.ctx.lib.msb_smooth_basis(self.ctx.h, self.h, op.h, int(max_sweeps),
                                           float(omega), float(tol), C.byref(n), C.byref(last),
                                           _ptr(deltas))
        self.ctx.check(st, "msb_smooth_basis")
        return n.value, last.value, deltas[:n.value], st

    # --- rows a4, a5
    def assemble(self, op: Operator):
        self.ctx.check(self.ctx.lib.msb_coarse_assemble(self.ctx.h, self.h, op.h),
                       "msb_coarse_assemble")

    def export(self, with_Ac=False):
        info = self.info()
        N, nnz, M = self.N, info["nnz"], info["M"]
        rowptr = np.empty(N + 1, dtype=np.int64)
        cols = np.empty(nnz, dtype=np.int32)
        vals = np.empty(nnz)
        Ac = np.empty((M, M)) if with_Ac else None
        self.ctx.check(self.ctx.lib.msb_level_export(self.ctx.h, self.h,
                                                     C.c_void_p(rowptr.ctypes.data),
                                                     _ptr(cols, np.int32), _ptr(vals),
                                                     _ptr(Ac) if Ac is not None else None),
                       "msb_level_export")
        return rowptr, cols, vals, Ac

    def export_coarse(self):
        """A_c of a Cartesian level as COO (rows, cols, vals) from its box-stencil storage."""
        nnz = C.c_int64()
        self.ctx.check(self.ctx.lib.msb_level_export_coarse(self.ctx.h, self.h, C.byref(nnz),
                                                            None, None, None),
                       "msb_level_export_coarse")
        r = np.empty(nnz.value, dtype=np.int32)
        c = np.empty(nnz.value, dtype=np.int32)
        v = np.empty(nnz.value)
        self.ctx.check(self.ctx.lib.msb_level_export_coarse(self.ctx.h, self.h, C.byref(nnz),
                                                            _ptr(r, np.int32), _ptr(c, np.int32),
                                                            _ptr(v)),
                       "msb_level_export_coarse")
        return r, c, v

    def import_values(self, vals):
        self.ctx.check(self.ctx.lib.msb_level_import_values(self.ctx.h, self.h, _ptr(vals)),
                       "msb_level_import_values")

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.msb_level_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Solver:
    """ms_iterate(b, tol) — rows a6–a11 (Eq. 8, Richardson, optional dynamic stage)."""

    SMOOTHERS = {"jacobi": 0, "ilu0": 1}

    def __init__(self, ctx: Context, op: Operator, levels: Sequence[Level], omega_s=2.0 / 3.0,
                 nu=1, post_smooth=False, dynamic=False, edges=(0.1, 0.5), max_blocks=1024,
                 smoother="jacobi"):
        self.ctx = ctx
        self.op = op
        self.levels = list(levels)
        arr = (C.c_void_p * max(1, len(self.levels)))(*[lv.h.value for lv in self.levels])
        h = C.c_void_p()
        ctx.check(ctx.lib.msb_solver_create(ctx.h, op.h, arr, len(self.levels), float(omega_s),
                                            int(nu), int(bool(post_smooth)), int(bool(dynamic)),
                                            float(edges[0]), float(edges[1]), int(max_blocks),
                                            C.byref(h)), "msb_solver_create")
        self.h = h
        if smoother != "jacobi":
            self.set_smoother(smoother)

    def set_smoother(self, smoother):
        """"jacobi" (damped, omega_s) or "ilu0" (red-black ILU(0), NEXT-2)."""
        self.ctx.check(self.ctx.lib.msb_solver_set_smoother(self.ctx.h, self.h,
                                                            self.SMOOTHERS[smoother]),
                       "msb_solver_set_smoother")

    def add_dynamic_basis(self, dp, part_out=None):
        M = C.c_int32()
        self.ctx.check(self.ctx.lib.msb_add_dynamic_basis(self.ctx.h, self.h, _ptr(dp), C.byref(M),
                                                          _ptr(part_out, np.int32)),
                       "msb_add_dynamic_basis")
        return M.value

    def iterate(self, x, b=None, tol=1e-6, max_iter=1000, fixed_iters=0, history=True):
        """x: in x0 / out x (torch CUDA tensor or numpy array).  Returns a dict."""
        n = C.c_int32()
        cap = max(max_iter, fixed_iters) + 2
        res = np.zeros(cap) if history else None
        dyn = np.zeros(cap, dtype=np.int32) if history else None
        st = self.ctx.lib.msb_ms_iterate(self.ctx.h, self.h, _ptr(b), _ptr(x), float(tol),
                                         int(max_iter), int(fixed_iters), C.byref(n),
                                         _ptr(res) if history else None,
                                         _ptr(dyn, np.int32) if history else None)
        self.ctx.check(st, "msb_ms_iterate")
        k = n.value
        out = dict(iters=k, status=st, converged=(st == OK and fixed_iters == 0))
        if history:
            out["res"] = res[:k + 1].copy()
            out["dyn_M"] = dyn[:k].copy()
        return out

    def fgmres(self, x, b=None, tol=1e-6, restart=20, max_iter=1000, fixed_iters=0):
        """Flexible GMRES right-preconditioned by one multibasis cycle (§8 NEXT-1).
        x: in x0 / out x.  Returns dict(iters, status, converged, res)."""
        n = C.c_int32()
        cap = max(max_iter, fixed_iters) + 2 + max(max_iter, fixed_iters) // max(1, restart) + 2
        res = np.zeros(cap)
        st = self.ctx.lib.msb_fgmres(self.ctx.h, self.h, _ptr(b), _ptr(x), float(tol), int(restart),
                                     int(max_iter), int(fixed_iters), C.byref(n), _ptr(res))
        self.ctx.check(st, "msb_fgmres")
        k = n.value
        return dict(iters=k, status=st, converged=(st == OK and fixed_iters == 0),
                    res=res[:k + 1].copy())

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.msb_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Cpr:
    """§8 NEXT-4: the CPR two-stage preconditioner of the compressible two-phase system
    (PAPER.md:122-203, :287-292).  `fluid`: a mapping with the msb_fluid fields."""

    METHODS = {"none": 0, "impes": 1, "quasi": 2}
    PRECONDS = {"cpr": 1, "ilu0": 2}

    def __init__(self, ctx: Context, op: Operator, level: Level, fluid, n_cycles=1,
                 omega_s=2.0 / 3.0):
        self.ctx = ctx
        self.op = op
        self.level = level  # kept alive: the CPR object reads its basis
        f = fluid if isinstance(fluid, dict) else vars(fluid)
        fl = L.Fluid(*[float(f[k]) for k in ("mu_w", "mu_o", "rho_w", "rho_o", "c_w", "c_o",
                                              "c_r", "phi", "p_ref", "dt")], int(f["nrel"]))
        h = C.c_void_p()
        ctx.check(ctx.lib.msb_cpr_create(ctx.h, op.h, level.h, C.byref(fl), int(n_cycles),
                                         float(omega_s), C.byref(h)), "msb_cpr_create")
        self.h = h
        self.N = op.N

    def linearize(self, p, S, p_n, S_n, q=None):
        self.ctx.check(self.ctx.lib.msb_cpr_linearize(self.ctx.h, self.h, _ptr(p), _ptr(S),
                                                      _ptr(p_n), _ptr(S_n), _ptr(q)),
                       "msb_cpr_linearize")

    def decouple(self, method="quasi"):
        self.ctx.check(self.ctx.lib.msb_cpr_decouple(self.ctx.h, self.h, self.METHODS[method]),
                       "msb_cpr_decouple")

    def apply(self, r, dx):
        self.ctx.check(self.ctx.lib.msb_cpr_apply(self.ctx.h, self.h, _ptr(r), _ptr(dx)),
                       "msb_cpr_apply")

    def apply_system(self, x, y):
        self.ctx.check(self.ctx.lib.msb_cpr_apply_system(self.ctx.h, self.h, _ptr(x), _ptr(y)),
                       "msb_cpr_apply_system")

    def export(self, decoupled=True):
        N = self.N
        F, J = np.empty(2 * N), np.empty(28 * N)
        w = Fs = Js = None
        if decoupled:
            w, Fs, Js = np.empty(2 * N), np.empty(2 * N), np.empty(14 * N)
        self.ctx.check(self.ctx.lib.msb_cpr_export(self.ctx.h, self.h, _ptr(F), _ptr(J), _ptr(w),
                                                   _ptr(Fs), _ptr(Js)), "msb_cpr_export")
        out = dict(F=F, J=J.reshape(2, 2, 7, N))
        if decoupled:
            out.update(w=w.reshape(2, N), Fs=Fs, Js=Js.reshape(2, 7, N))
        return out

    def export_coarse(self):
        M = C.c_int32()
        self.ctx.check(self.ctx.lib.msb_cpr_export_coarse(self.ctx.h, self.h, None, C.byref(M)),
                       "msb_cpr_export_coarse")
        Ac = np.empty(M.value * M.value)
        self.ctx.check(self.ctx.lib.msb_cpr_export_coarse(self.ctx.h, self.h, _ptr(Ac),
                                                          C.byref(M)), "msb_cpr_export_coarse")
        return Ac.reshape(M.value, M.value)

    def fgmres(self, x, b=None, tol=1e-8, restart=40, max_iter=200, fixed_iters=0,
               precond="cpr"):
        n = C.c_int32()
        cap = max(max_iter, fixed_iters) + 2 + max(max_iter, fixed_iters) // max(1, restart) + 2
        res = np.zeros(cap)
        st = self.ctx.lib.msb_cpr_fgmres(self.ctx.h, self.h, _ptr(b), _ptr(x), float(tol),
                                         int(restart), int(max_iter), int(fixed_iters),
                                         self.PRECONDS[precond], C.byref(n), _ptr(res))
        self.ctx.check(st, "msb_cpr_fgmres")
        k = n.value
        return dict(iters=k, status=st, converged=(st == OK and fixed_iters == 0),
                    res=res[:k + 1].copy())

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.msb_cpr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
