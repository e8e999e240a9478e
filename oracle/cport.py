"""ctypes wrapper of oracle/librto.so (C + OpenMP restatement) -- TEST / CPU-BASELINE ONLY."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_LIB = None
PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "librto.so")
FS = {"ie": 0, "exp_linear": 1, "exp_parabolic": 2}


def lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(PATH)
        d = ctypes.POINTER(ctypes.c_double)
        _LIB.rto_apply_A_slab.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int] + \
            [d] * 11 + [ctypes.c_int]
        _LIB.rto_apply_A_slab.restype = ctypes.c_int
        _LIB.rto_max_threads.restype = ctypes.c_int
    return _LIB


def max_threads() -> int:
    return int(lib().rto_max_threads())


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class SlabPort:
    """Holds contiguous copies of a SlabDesc's arrays (gamma must be mu-independent)."""

    def __init__(self, desc):
        g = np.asarray(desc.gamma).reshape(desc.n_space, desc.n_angles, desc.n_freq)
        if not np.all(g == g[:, :1, :]):
            raise ValueError("C port supports mu-independent gamma only")
        self.d = desc
        self.arrs = [np.ascontiguousarray(a, dtype=float) for a in
                     (desc.t_nodes, desc.mu, desc.ang_w, desc.phi, desc.freq_w, desc.ybasis, desc.coeffs, desc.R,
                      g[:, 0, :])]

    def apply_A(self, x, y=None, nthreads: int = 0):
        d = self.d
        x = np.ascontiguousarray(x, dtype=float)
        if y is None:
            y = np.empty_like(x)
        rc = lib().rto_apply_A_slab(d.n_space, d.n_angles, d.n_freq, d.ybasis.shape[0], FS[d.formal_solver],
                                    *[_p(a) for a in self.arrs], _p(x), _p(y), nthreads)
        if rc:
            raise MemoryError("rto_apply_A_slab allocation failed")
        return y
