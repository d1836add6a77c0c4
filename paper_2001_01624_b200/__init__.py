"""B200-native MsRSB basis smoothing + iterative multiscale multibasis pressure cycle.

Hot path of Klemetsdal, Møyner & Lie, arXiv 2001.01624, as hand-written sm_100a
CUDA kernels behind the C ABI in include/msb.h (libmsb.so, built in-tree), with
this thin ctypes binding.  PyTorch supplies device memory and streams only.
"""
from .api import (Context, Cpr, Level, MsbError, Operator, Solver,  # noqa: F401
                  partition_cartesian)
from . import _lib  # noqa: F401

__all__ = ["Context", "Operator", "Level", "Solver", "Cpr", "MsbError", "partition_cartesian"]
