"""ORACLE (test infrastructure only; see oracle/__init__.py).

ctypes loader for the plain C fp64 cell-list oracle (oracle/celllist.c).
__graft_entry__.build() compiles it; `ensure_built()` compiles on demand with gcc
(-O2 -fopenmp -ffp-contract=off: no FMA contraction in the fp32 cell-index
contract).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import reference as ref

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "celllist.c")
_LIB = os.path.join(_HERE, "_celllist.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        _lib.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib.oracle_set_threads.restype = ctypes.c_int
        _lib.oracle_cells.argtypes = [ctypes.c_int64, P, P, P, P, ctypes.c_float, P, P]
        _lib.oracle_bin.argtypes = [ctypes.c_int64, P, ctypes.c_int64, P, P, P]
        _lib.oracle_interact.argtypes = [ctypes.c_int64, P, P, P, P, P, ctypes.c_float, P, ctypes.c_double,
                                         P, ctypes.c_int, ctypes.c_double, ctypes.c_int64, P,
                                         P, P, P, P, P]
    return _lib


def set_threads(n: int = 0) -> int:
    """Set the OpenMP thread count (n <= 0: keep); returns the count in use."""
    return int(_load().oracle_set_threads(int(n)))


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _geom(grid):
    o = np.array(grid.origin, dtype=np.float32)
    d = np.array(grid.dims, dtype=np.int32)
    return o, ref.inv_width(grid), d


def cells(x, y, z, grid) -> np.ndarray:
    lib = _load()
    x, y, z = (np.ascontiguousarray(a, np.float32) for a in (x, y, z))
    o, inv_w, d = _geom(grid)
    out = np.empty(len(x), np.int64)
    lib.oracle_cells(len(x), _p(x), _p(y), _p(z), _p(o), inv_w, _p(d), _p(out))
    return out


def binning(cell, ncells):
    lib = _load()
    cell = np.ascontiguousarray(cell, np.int64)
    counts = np.empty(ncells, np.int64)
    offsets = np.empty(ncells + 1, np.int64)
    order = np.empty(len(cell), np.int64)
    lib.oracle_bin(len(cell), _p(cell), ncells, _p(counts), _p(offsets), _p(order))
    return counts, offsets, order


def interact(x, y, z, q, grid, kernel=ref.KERNEL_GAUSSIAN, targets=None, band=None, threads=None):
    """Cell-list fp64 oracle; `targets` = indices (into the input arrays) to evaluate (default all)."""
    lib = _load()
    x, y, z, q = (np.ascontiguousarray(a, np.float32) for a in (x, y, z, q))
    o, inv_w, d = _geom(grid)
    if band is None:
        band = ref.band_rel(grid)
    if targets is None:
        nt, tp = len(x), None
    else:
        targets = np.ascontiguousarray(targets, np.int64)
        nt, tp = len(targets), _p(targets)
    out = np.empty((nt, 4))
    S = np.empty((nt, 4))
    A = np.empty((nt, 4))
    C = np.empty(nt, np.int64)
    P = np.empty(nt, np.int64)
    if threads is not None:
        set_threads(threads)
    kp = np.array([float(np.float32(grid.sig)), *ref.lj_params(grid)], dtype=np.float64)
    lib.oracle_interact(len(x), _p(x), _p(y), _p(z), _p(q), _p(o), inv_w, _p(d), float(np.float32(grid.r_c)),
                        _p(kp), int(kernel), float(band), nt, tp, _p(out), _p(S), _p(A), _p(C), _p(P))
    return dict(out=out, S=S, A=A, C=C, P=P)
