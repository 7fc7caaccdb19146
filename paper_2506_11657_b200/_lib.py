"""ctypes declarations of include/tem_b200.h (argument marshalling only).

Loading fails loudly: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os

from . import build as _build

_LIB = None


class SolveStats(ctypes.Structure):
    _fields_ = [("loop_ms", ctypes.c_double), ("kernel_launches", ctypes.c_longlong),
                ("shift_iterations", ctypes.c_longlong), ("iterations", ctypes.c_int),
                ("grid", ctypes.c_int), ("block", ctypes.c_int), ("real_shifts", ctypes.c_int),
                ("persistent", ctypes.c_int)]


class ForwardOpts(ctypes.Structure):
    """tem_forward_opts (include/tem_b200.h)."""
    _fields_ = [("tol", ctypes.c_double), ("maxit", ctypes.c_int), ("max_refine", ctypes.c_int),
                ("refine_tol", ctypes.c_double), ("channel_tol", ctypes.c_double), ("safety", ctypes.c_double)]


class ForwardStats(ctypes.Structure):
    """tem_forward_stats (include/tem_b200.h)."""
    _fields_ = [("refine_rounds", ctypes.c_int), ("shift_iterations", ctypes.c_longlong),
                ("initial_shift_iterations", ctypes.c_longlong), ("loop_ms", ctypes.c_double),
                ("channel_bound", ctypes.c_double), ("relres_max", ctypes.c_double),
                ("kernel_launches", ctypes.c_longlong)]


_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)

SIGNATURES = {
    "tem_version": ([], ctypes.c_char_p),
    "tem_last_error": ([], ctypes.c_char_p),
    "tem_create": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, _D, _D, _D, ctypes.POINTER(_P)], ctypes.c_int),
    "tem_destroy": ([_P], None),
    "tem_num_nodes": ([_P], ctypes.c_size_t),
    "tem_num_unknowns": ([_P], ctypes.c_size_t),
    "tem_edge_mass": ([_P, _P, _P, _P], ctypes.c_int),
    "tem_apply_shifted": ([_P, _P, ctypes.c_int, _D, _P, _P, _P], ctypes.c_int),
    "tem_cocg_workspace_bytes": ([_P, ctypes.c_int], ctypes.c_size_t),
    "tem_cocg_solve": ([_P, _P, _P, ctypes.c_int, _D, ctypes.c_double, ctypes.c_int, _P, _P,
                        ctypes.c_size_t, _I, _D, _P], ctypes.c_int),
    "tem_last_solve_stats": ([_P, ctypes.POINTER(SolveStats)], ctypes.c_int),
    "tem_set_solver": ([_P, ctypes.c_int], ctypes.c_int),
    "tem_get_solver": ([_P], ctypes.c_int),
    "tem_set_launch_mode": ([_P, ctypes.c_int], ctypes.c_int),
    "tem_get_launch_mode": ([_P], ctypes.c_int),
    "tem_synthesize": ([_P, ctypes.c_int, ctypes.c_int, _D, _I, _P, _P, _P], ctypes.c_int),
    "tem_curl_z": ([_P, ctypes.c_int, _P, ctypes.c_int, _I, _P, _P], ctypes.c_int),
    "tem_cocg_solve_rhs": ([_P, _P, _P, ctypes.c_int, _D, _D, ctypes.c_int, _P, _P, ctypes.c_size_t, _I,
                            _D, _P], ctypes.c_int),
    "tem_forward_default_opts": ([ctypes.POINTER(ForwardOpts)], None),
    "tem_forward_workspace_bytes": ([_P, ctypes.c_int, ctypes.c_int], ctypes.c_size_t),
    "tem_forward": ([_P, _P, _P, ctypes.c_int, _D, ctypes.c_int, _D, _I, ctypes.POINTER(ForwardOpts), _P, _P,
                     _P, ctypes.c_size_t, _I, _D, ctypes.POINTER(ForwardStats), _P], ctypes.c_int),
    "tem_residual": ([_P, _P, _P, ctypes.c_int, _D, _P, _P, _D, _P], ctypes.c_int),
    "tem_last_forward_stats": ([_P, ctypes.POINTER(ForwardStats)], ctypes.c_int),
    "tem_forward_host": ([_P, _D, _D, ctypes.c_int, _D, ctypes.c_int, _D, _I, ctypes.POINTER(ForwardOpts),
                          _D, _I, _D], ctypes.c_int),
    "tem_fit_family": ([ctypes.c_int, _D, _D, ctypes.c_int, ctypes.c_int, _I, _D, _D, _I, _D],
                       ctypes.c_int),
}


def lib_path() -> str:
    """The in-tree library; TEM_LIB overrides it (build-variant experiments)."""
    return os.environ.get("TEM_LIB") or _build.LIB


def load(build_if_missing: bool = True):
    """Load libtem_b200.so (building it with nvcc if absent)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        if not build_if_missing:
            raise ImportError(f"{path} missing: run `python -m paper_2506_11657_b200.build`")
        _build.build()
    lib = ctypes.CDLL(path)
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None and os.environ.get("TEM_LIB"):   # an older build variant (experiments)
            continue
        if fn is None:
            raise ImportError(f"{path} does not export {name}")
        fn.argtypes = args
        fn.restype = res
    _LIB = lib
    return lib


class TemError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"tem_b200 error {code}: {msg}")
        self.code = code


TEM_ENOCONV = -4
TEM_EBREAKDOWN = -5


def check(rc: int):
    if rc != 0:
        raise TemError(rc, load().tem_last_error().decode())
