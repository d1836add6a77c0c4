"""ctypes declarations of include/msb.h.  Loads the in-tree libmsb.so and fails
loudly if it is missing or cannot be loaded — there is no fallback."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmsb.so")


class Grid(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
                ("dx", C.c_double), ("dy", C.c_double), ("dz", C.c_double)]


class Source(C.Structure):
    _fields_ = [("cell", C.c_int32), ("rate", C.c_double)]


class Fluid(C.Structure):
    _fields_ = [("mu_w", C.c_double), ("mu_o", C.c_double), ("rho_w", C.c_double),
                ("rho_o", C.c_double), ("c_w", C.c_double), ("c_o", C.c_double),
                ("c_r", C.c_double), ("phi", C.c_double), ("p_ref", C.c_double),
                ("dt", C.c_double), ("nrel", C.c_int32)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)

p = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f64 = C.c_double
pi32 = C.POINTER(C.c_int32)
pi64 = C.POINTER(C.c_int64)
pf64 = C.POINTER(C.c_double)

# name: (restype, argtypes)
SIGNATURES = {
    "msb_ctx_create": (i32, [C.POINTER(p), C.c_int, p, ALLOC_FN, FREE_FN, p]),
    "msb_ctx_destroy": (i32, [p]),
    "msb_ctx_set_stream": (i32, [p, p]),
    "msb_last_error": (C.c_char_p, [p]),
    "msb_version": (C.c_char_p, []),
    "msb_launch_count": (i64, []),
    "msb_build_tpfa": (i32, [p, C.POINTER(Grid), p, p, p, C.POINTER(Source), i32, C.POINTER(p)]),
    "msb_op_set_mobility": (i32, [p, p, p]),
    "msb_op_export": (i32, [p, p, p, p]),
    "msb_op_apply": (i32, [p, p, p, p]),
    "msb_op_destroy": (i32, [p]),
    "msb_partition_cartesian": (i32, [p, C.POINTER(Grid), i32, i32, i32, p, pi32]),
    "msb_level_create_cartesian": (i32, [p, p, i32, i32, i32, C.POINTER(p), pi64]),
    "msb_level_create_split": (i32, [p, p, p, C.POINTER(p), pi64]),
    "msb_level_create_constant": (i32, [p, p, p, i32, C.POINTER(p)]),
    "msb_solver_set_smoother": (i32, [p, p, i32]),
    "msb_partition_wells": (i32, [p, C.POINTER(Grid), p, p, i32, i32, p, pi32]),
    "msb_partition_indicator": (i32, [p, p, p, p, i32, i32, p, pi32]),
    "msb_level_create_general": (i32, [p, p, p, i32, i32, C.POINTER(p), pi64]),
    "msb_level_info": (i32, [p, p, pi32, pi64, pi32, p]),
    "msb_level_export": (i32, [p, p, p, p, p, p]),
    "msb_level_import_values": (i32, [p, p, p]),
    "msb_level_export_coarse": (i32, [p, p, pi64, p, p, p]),
    "msb_level_destroy": (i32, [p]),
    "msb_smooth_basis": (i32, [p, p, p, i32, f64, f64, pi32, pf64, p]),
    "msb_coarse_assemble": (i32, [p, p, p]),
    "msb_solver_create": (i32, [p, p, C.POINTER(p), i32, f64, i32, i32, i32, f64, f64, i32,
                                C.POINTER(p)]),
    "msb_add_dynamic_basis": (i32, [p, p, p, pi32, p]),
    "msb_ms_iterate": (i32, [p, p, p, p, f64, i32, i32, pi32, p, p]),
    "msb_solver_destroy": (i32, [p]),
    "msb_fgmres": (i32, [p, p, p, p, f64, i32, i32, i32, pi32, p]),
    "msb_transport_upwind": (i32, [p, p, p, p, p, f64, f64, f64, p, pi32]),
    "msb_upstream_mobility": (i32, [p, p, p, p, f64, f64, p]),
    "msb_transport_step_size": (i32, [p, p, p, f64, pf64]),
    "msb_cpr_create": (i32, [p, p, p, C.POINTER(Fluid), i32, f64, C.POINTER(p)]),
    "msb_cpr_linearize": (i32, [p, p, p, p, p, p, p]),
    "msb_cpr_decouple": (i32, [p, p, i32]),
    "msb_cpr_apply": (i32, [p, p, p, p]),
    "msb_cpr_apply_system": (i32, [p, p, p, p]),
    "msb_cpr_export": (i32, [p, p, p, p, p, p, p]),
    "msb_cpr_export_coarse": (i32, [p, p, p, pi32]),
    "msb_cpr_fgmres": (i32, [p, p, p, p, f64, i32, i32, i32, i32, pi32, p]),
    "msb_cpr_destroy": (i32, [p]),
}

_lib = None


def load():
    """Load libmsb.so (raises if absent: the CUDA path is the only path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libmsb.so not built at {LIB_PATH}; run __graft_entry__.build()")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
