"""ctypes binding of libpi.so (include/pi.h).  Argument marshalling only: every step of the
hot path runs in the library's CUDA kernels.  There is no CPU fallback: if the shared library
is missing, importing this module raises."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIBPATH = os.path.join(HERE, "libpi.so")

PI_OK, PI_EINVAL, PI_ECAPACITY, PI_EINAPPLICABLE, PI_ECUDA, PI_ENCCL, PI_ESTATE, PI_EDEVICE = range(8)
STATUS_NAMES = ["PI_OK", "PI_EINVAL", "PI_ECAPACITY", "PI_EINAPPLICABLE", "PI_ECUDA", "PI_ENCCL", "PI_ESTATE",
                "PI_EDEVICE"]
KERNELS = {"gaussian": 0, "indicator": 1, "candidate": 2, "lj": 3, "lowflop": 4, "highflop": 5}
ALGOS = {"global": 0, "fullload": 1, "xpencil": 2, "auto": 3, "xpreg": 4, "half": 5}


class pi_config(ctypes.Structure):
    _fields_ = [("origin", ctypes.c_float * 3), ("cell_width", ctypes.c_float), ("dims", ctypes.c_int32 * 3),
                ("r_c", ctypes.c_float), ("kernel", ctypes.c_int32), ("kparam", ctypes.c_float * 4),
                ("capacity", ctypes.c_int64), ("stream", ctypes.c_void_p), ("rank", ctypes.c_int32),
                ("nranks", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p), ("x_subcells", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 7)]


class pi_stats(ctypes.Structure):
    _fields_ = [("n_owned", ctypes.c_int64), ("n_ghost", ctypes.c_int64), ("max_per_cell", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("candidates", ctypes.c_int64), ("fallback_cells", ctypes.c_int64),
                ("migrants_in", ctypes.c_int64), ("migrants_out", ctypes.c_int64), ("steps", ctypes.c_int64),
                ("exchange_bytes", ctypes.c_int64), ("phase_ms", ctypes.c_double * 4),
                ("overlapped_steps", ctypes.c_int64), ("reserved", ctypes.c_int64 * 2)]


class pi_tuning(ctypes.Structure):
    _fields_ = [("xpencil_len", ctypes.c_int32), ("xpencil_cap", ctypes.c_int32),
                ("fullload_box", ctypes.c_int32 * 3), ("fullload_cap", ctypes.c_int32), ("threads", ctypes.c_int32),
                ("xpencil_slots", ctypes.c_int32), ("xpencil_targets", ctypes.c_int32),
                ("exchange_full", ctypes.c_int32), ("xpencil_layout", ctypes.c_int32),
                ("exchange_overlap", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3)]


P = ctypes.c_void_p
SIGNATURES = {
    "pi_abi_version": (ctypes.c_int32, []),
    "pi_workspace_bytes": (ctypes.c_size_t, [ctypes.POINTER(pi_config)]),
    "pi_slab_info": (ctypes.c_int, [ctypes.POINTER(pi_config), ctypes.POINTER(ctypes.c_int64)]),
    "pi_nccl_unique_id": (ctypes.c_int, [P]),
    "pi_create": (ctypes.c_int, [ctypes.POINTER(pi_config), P, ctypes.c_size_t, ctypes.POINTER(P)]),
    "pi_destroy": (ctypes.c_int, [P]),
    "pi_set_stream": (ctypes.c_int, [P, P]),
    "pi_set_tuning": (ctypes.c_int, [P, ctypes.POINTER(pi_tuning)]),
    "pi_bin": (ctypes.c_int, [P, ctypes.c_int64, P, P, P, P, P]),
    "pi_interact": (ctypes.c_int, [P, ctypes.c_int, P, P, P, P]),
    "pi_step": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_float]),
    "pi_run_host": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int64, P, P, P, P, P, P, P, P]),
    "pi_run_host_submit": (ctypes.c_int, [P, ctypes.c_int, ctypes.c_int64, P, P, P, P, P, P, P, P]),
    "pi_run_host_wait": (ctypes.c_int, [P]),
    "pi_get_binning": (ctypes.c_int, [P, P, P, P, P]),
    "pi_get_particles": (ctypes.c_int, [P, P, P, P, P, P, P, P, P, P]),
    "pi_get_stats": (ctypes.c_int, [P, ctypes.POINTER(pi_stats)]),
    "pi_count_pairs": (ctypes.c_int, [P, ctypes.POINTER(ctypes.c_int64)]),
    "pi_last_error": (ctypes.c_char_p, [P]),
}

_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIBPATH):
        raise ImportError(f"libpi.so not built ({LIBPATH}); run `python -c 'import __graft_entry__ as g; g.build()'` "
                          "or `python paper_2406_16091_b200/build.py` (nvcc, sm_100a).  There is no CPU fallback.")
    lib = ctypes.CDLL(LIBPATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib
