"""ctypes binding of ``libpgx.so`` (the C ABI declared in ``include/pgx.h``).

The library is built in-tree by ``paper_2605_20816_b200.build.build_library``
(``__graft_entry__.build()``).  There is no CPU fallback: if the library or a
CUDA device is missing every hot-path call raises.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_int64, c_size_t, c_uint32, c_void_p

from .errors import NumericalError, ResourceError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")
# PGX_LIB: an alternative in-tree build (A/B kernel experiments, tools/)
LIB_PATH = os.environ.get("PGX_LIB") or os.path.join(LIB_DIR, "libpgx.so")

PGX_OK = 0
PGX_ERR_INVALID_ARGUMENT = 1
PGX_ERR_RESOURCE = 2
PGX_ERR_NUMERICAL = 3
PGX_ERR_CUDA = 4

PGX_BASIS_MONOMIAL = 0
PGX_BASIS_LEGENDRE = 1

PGX_PREC_EXACT = 0
PGX_PREC_FP64 = 1
PGX_PREC_TC = 2
PRECISIONS = {"exact": PGX_PREC_EXACT, "fp64": PGX_PREC_FP64, "tc": PGX_PREC_TC}

PGX_WANT_GRAD = 1
PGX_WANT_ASSIGN = 2
PGX_DEVICE_PTRS = 4
PGX_THETA_F32 = 8

PGX_STAT_RANGE = 1  # pgx_stats.flags: theta beyond the fast modes' logit range
PGX_FAST_RANGE = 65536.0
ABI_VERSION = 2
STATS_WORDS = 9  # sizeof(pgx_stats) / 8

PGX_PATH_GENERAL = 0
PGX_PATH_GRID_FP64 = 1
PGX_PATH_GRID_TC = 2
PATH_NAMES = {PGX_PATH_GENERAL: "general", PGX_PATH_GRID_FP64: "grid_fp64", PGX_PATH_GRID_TC: "grid_tc"}

PGX_MEM_HOST = 0
PGX_MEM_DEVICE = 1


class PgxDesc(ctypes.Structure):
    _fields_ = [
        ("dim", c_int32),
        ("basis_kind", c_int32),
        ("degree", c_int32),
        ("n_grains", c_int32),
        ("n_points", c_int64),
        ("resolution", c_int32),
        ("precision", c_int32),
        ("points", c_void_p),
        ("labels0", c_void_p),
        ("mem", c_int32),
        ("device", c_int32),
        ("stream", c_void_p),
        ("design", c_void_p),
        ("design_k", c_int32),
    ]


class PgxStats(ctypes.Structure):
    _fields_ = [
        ("phi", c_double),
        ("err", c_double),
        ("e0", c_double),
        ("n_rescanned", c_double),
        ("n_points", c_int64),
        ("n_correct", c_int64),
        ("n_ambiguous", c_int64),
        ("n_nonfinite", c_int64),
        ("flags", c_int64),
    ]


# Every symbol include/pgx.h declares, with its ctypes signature.
SIGNATURES = {
    "pgx_abi_version": (c_int, []),
    "pgx_last_error": (c_char_p, []),
    "pgx_workspace_bytes": (c_size_t, [POINTER(PgxDesc)]),
    "pgx_problem_create": (c_int, [POINTER(PgxDesc), POINTER(c_void_p)]),
    "pgx_problem_destroy": (None, [c_void_p]),
    "pgx_set_stream": (c_int, [c_void_p, c_void_p]),
    "pgx_eval": (c_int, [c_void_p, c_void_p, c_double, c_double, c_uint32, c_void_p, c_void_p]),
    "pgx_assign": (c_int, [c_void_p, c_void_p, c_uint32, c_void_p, c_void_p, c_void_p]),
    "pgx_lbfgs_create": (c_int, [c_void_p, c_int, ctypes.POINTER(c_void_p)]),
    "pgx_lbfgs_destroy": (None, [c_void_p]),
    "pgx_lbfgs_start": (c_int, [c_void_p, c_void_p, c_double, c_double, c_void_p]),
    "pgx_lbfgs_restart": (c_int, [c_void_p, c_double, c_double, c_void_p]),
    "pgx_lbfgs_clear": (c_int, [c_void_p]),
    "pgx_lbfgs_direction": (c_int, [c_void_p, c_int, c_void_p]),
    "pgx_lbfgs_trial": (c_int, [c_void_p, c_double, c_double, c_double, c_void_p]),
    "pgx_lbfgs_accept": (c_int, [c_void_p, c_int, c_void_p]),
    "pgx_lbfgs_theta": (c_int, [c_void_p, c_void_p]),
    "pgx_lbfgs_iterate": (c_int, [c_void_p, c_int, c_double, c_double, c_double, c_void_p]),
    "pgx_last_launch_count": (c_int, [c_void_p]),
    "pgx_problem_path": (c_int, [c_void_p]),
    "pgx_set_profiling": (c_int, [c_void_p, c_int]),
    "pgx_profile_count": (c_int, [c_void_p]),
    "pgx_profile_name": (c_char_p, [c_void_p, c_int]),
    "pgx_profile_ms": (c_float, [c_void_p, c_int]),
    "pgx_synchronize": (c_int, [c_void_p]),
    "pgx_soft_assign": (c_int, [c_void_p, c_void_p, c_double, c_uint32, c_void_p]),
    "pgx_label_moments": (c_int, [c_int, ctypes.c_int64, c_void_p, c_int, c_void_p]),
    "pgx_label_moments_error": (c_char_p, []),
    "pgx_problem_label_moments": (c_int, [c_void_p, c_uint32, c_void_p]),
    "pgx_problem_bytes": (c_size_t, [c_void_p]),
}

_lib = None


def load():
    """Load libpgx.so once; raise loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: the pgx hot path has no CPU fallback. "
            "Build it with `python -c 'import __graft_entry__ as g; g.build()'`.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (restype, argtypes) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    if lib.pgx_abi_version() != ABI_VERSION:
        raise RuntimeError("libpgx.so ABI version mismatch")
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().pgx_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    """Map a pgx_status onto the reference's exception types (errors.py:4-13)."""
    if status == PGX_OK:
        return
    msg = last_error()
    if status == PGX_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == PGX_ERR_RESOURCE:
        raise ResourceError(msg)
    if status == PGX_ERR_NUMERICAL:
        raise NumericalError(msg)
    raise RuntimeError(f"pgx CUDA error: {msg}")


def as_ptr(arr) -> int:
    return arr.ctypes.data if arr is not None else 0


__all__ = [n for n in dir() if n.startswith(("PGX_", "Pgx", "PREC"))] + [
    "load", "check", "last_error", "LIB_PATH", "SIGNATURES", "as_ptr", "c_float"]
