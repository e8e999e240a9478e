"""ctypes binding of librtk_b200.so (include/rtk_b200.h).

The shared library is built in-tree by ``python __graft_entry__.py`` /
``make -C paper_2602_21958_b200/csrc``.  There is no fallback: if the library
or a CUDA device is missing, every operator call raises.
"""

from __future__ import annotations

import ctypes
import os

from paper_2602_21958_b200.errors import ResourceLimitError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "librtk_b200.so")

RTK_OK, RTK_EINVAL, RTK_ERESOURCE, RTK_ECUDA = 0, 1, 2, 3
FS_CODES = {"ie": 0, "exp_linear": 1, "exp_parabolic": 2}
MAX_MOMENTS = 8

c_double_p = ctypes.POINTER(ctypes.c_double)


class SlabDesc(ctypes.Structure):
    _fields_ = [
        ("n_space", ctypes.c_int64),
        ("n_angles", ctypes.c_int32),
        ("n_freq", ctypes.c_int32),
        ("n_moments", ctypes.c_int32),
        ("formal_solver", ctypes.c_int32),
        ("gamma_per_ray", ctypes.c_int32),
        ("layout", ctypes.c_int32),
        ("t_nodes", c_double_p),
        ("mu", c_double_p),
        ("ang_w", c_double_p),
        ("phi", c_double_p),
        ("freq_w", c_double_p),
        ("ybasis", c_double_p),
        ("coeffs", c_double_p),
        ("redistribution", c_double_p),
        ("gamma", c_double_p),
        ("inflow", c_double_p),
    ]


class SolveCfg(ctypes.Structure):
    _fields_ = [
        ("rel_tol", ctypes.c_double),
        ("max_iter", ctypes.c_int32),
        ("restart", ctypes.c_int32),
        ("reorthogonalize", ctypes.c_int32),
        ("orthogonalization", ctypes.c_int32),
    ]


class SolveRep(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("converged", ctypes.c_int32),
        ("breakdown", ctypes.c_int32),
        ("n_history", ctypes.c_int32),
        ("true_residual", ctypes.c_double),
        ("matvecs", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


MATVEC_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_int64, ctypes.c_void_p)

# (name, restype, argtypes) for every symbol of include/rtk_b200.h
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
SIGNATURES = [
    ("rtk_last_error_message", ctypes.c_char_p, []),
    ("rtk_version", ctypes.c_int, []),
    ("rtk_kernel_launch_count", _I64, []),
    ("rtk_problem_create_slab", ctypes.c_int, [ctypes.POINTER(SlabDesc), ctypes.POINTER(_P)]),
    ("rtk_problem_create_lattice", ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    ("rtk_problem_destroy", ctypes.c_int, [_P]),
    ("rtk_problem_n_total", _I64, [_P]),
    ("rtk_problem_set_inflow", ctypes.c_int, [_P, _P, _I64, _P]),
    ("rtk_problem_set_tuning", ctypes.c_int, [_P, ctypes.c_char_p, _I64]),
    ("rtk_apply_A", ctypes.c_int, [_P, _P, _P, _I64, _P]),
    ("rtk_apply_A_host", ctypes.c_int, [_P, _P, _P, _I64, _P]),
    ("rtk_apply_A_host_batch", ctypes.c_int, [_P, _P, _P, _I32, _I64]),
    ("rtk_profile_apply_A", ctypes.c_int, [_P, _P, _P, _I64, _P, ctypes.POINTER(ctypes.c_float)]),
    ("rtk_intensity_from_moments", ctypes.c_int, [_P, _P, _P, _P, _I64, _P]),
    ("rtk_partial_moments", ctypes.c_int, [_P, _P, _P, _I64, _P]),
    ("rtk_apply_A_with_moments", ctypes.c_int, [_P, _P, _P, _I64, _P, _I64, _P]),
    ("rtk_lattice_partial_moments", ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _P]),
    ("rtk_lattice_apply_with_moments", ctypes.c_int, [_P, _P, _P, _I64, _P, _I64, _P]),
    ("rtk_lattice_apply_with_moments_nodes", ctypes.c_int, [_P, _P, _P, _I64, _I64, _P, _P]),
    ("rtk_apply_sigma", ctypes.c_int, [_P, _P, _P, _I64, _P]),
    ("rtk_apply_lambda", ctypes.c_int, [_P, _P, _P, _I64, _P]),
    ("rtk_boundary", ctypes.c_int, [_P, _P, _I64, _P]),
    ("rtk_build_rhs", ctypes.c_int, [_P, _P, _P, _I64, _I32, _P]),
    ("rtk_source_function", ctypes.c_int, [_P, _P, _P, _P, _I64, _P]),
    ("rtk_gmres", ctypes.c_int, [MATVEC_FN, _P, _I64, _P, _P, ctypes.POINTER(SolveCfg), ctypes.POINTER(SolveRep),
                                 _P, _I32, _P]),
    ("rtk_gmres_problem", ctypes.c_int, [_P, _P, _P, ctypes.POINTER(SolveCfg), ctypes.POINTER(SolveRep), _P, _I32,
                                         _P]),
    ("rtk_bicgstab", ctypes.c_int, [MATVEC_FN, _P, _I64, _P, _P, ctypes.POINTER(SolveCfg),
                                    ctypes.POINTER(SolveRep), _P, _I32, _P]),
    ("rtk_problem_matvec", ctypes.c_int, [_P, _P, _P, _I64, _P]),
    ("rtk_dot", ctypes.c_int, [_P, _P, _I64, _P, _P]),
    ("rtk_block_dot", ctypes.c_int, [_P, _I32, _P, _I64, _P, _P]),
]

_lib = None


class NativeLibraryError(RuntimeError):
    """librtk_b200.so is missing or unusable (no CPU fallback exists)."""


def lib():
    """Load (once) and return the ctypes handle with typed signatures."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        handle = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    """Map C status codes to the reference's exception types."""
    if rc == RTK_OK:
        return
    msg = lib().rtk_last_error_message().decode(errors="replace")
    if rc == RTK_EINVAL:
        raise ValueError(msg)
    if rc == RTK_ERESOURCE:
        raise ResourceLimitError(msg)
    raise RuntimeError(f"CUDA failure in librtk_b200: {msg}")


def launch_count() -> int:
    return int(lib().rtk_kernel_launch_count())
