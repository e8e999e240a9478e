"""Device-vector plumbing: numpy <-> torch CUDA tensors, streams, handles.

torch is used only for device memory and the current CUDA stream; every
computation is a librtk_b200 kernel.  numpy inputs are copied to the device
and results copied back (the reference's calling convention); torch CUDA
float64 tensors are used zero-copy and results are returned as tensors.
"""

from __future__ import annotations

import ctypes

import numpy as np

from paper_2602_21958_b200 import _native


def _torch():
    import torch

    return torch


def require_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_21958_b200 needs a CUDA device (B200); there is no CPU fallback")
    _native.lib()
    return torch


def is_tensor(v) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(v, torch.Tensor)


def to_device(v, n: int):
    """Return (cuda float64 contiguous tensor, kind) for a numpy array or tensor."""
    torch = require_cuda()
    if isinstance(v, torch.Tensor):
        t = v.reshape(-1)
        if t.numel() != n:
            raise ValueError(f"expected length {n}, got {t.numel()}")
        if not t.is_cuda:
            return t.to(device="cuda", dtype=torch.float64).contiguous(), "cpu_tensor"
        if t.dtype != torch.float64 or not t.is_contiguous():
            t = t.to(torch.float64).contiguous()
        return t, "cuda"
    arr = np.ascontiguousarray(np.asarray(v, dtype=float).reshape(-1))
    if arr.size != n:
        raise ValueError(f"expected length {n}, got {arr.size}")
    return torch.from_numpy(arr).to("cuda"), "numpy"


def from_device(t, kind):
    if kind == "numpy":
        return t.cpu().numpy()
    if kind == "cpu_tensor":
        return t.cpu()
    return t


def empty(n: int):
    torch = require_cuda()
    return torch.empty(n, dtype=torch.float64, device="cuda")


def stream_ptr():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_native.c_double_p)


class _CudaView:
    """__cuda_array_interface__ wrapper so torch.as_tensor can view a raw device pointer."""

    def __init__(self, address: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (address, False),
                                         "version": 3, "strides": None}


def view(address: int, n: int):
    torch = _torch()
    return torch.as_tensor(_CudaView(address, n), device="cuda")


class SlabHandle:
    """Owns one rtk_problem (device-resident tables + workspace)."""

    def __init__(self, arrays: dict, formal_solver: str, gamma_per_ray: bool, n_space: int, n_angles: int,
                 n_freq: int, n_moments: int, layout: str = "intensity"):
        require_cuda()
        lib = _native.lib()
        self._keep = {k: np.ascontiguousarray(v, dtype=float) for k, v in arrays.items() if v is not None}
        d = _native.SlabDesc()
        d.n_space, d.n_angles, d.n_freq, d.n_moments = n_space, n_angles, n_freq, n_moments
        if formal_solver not in _native.FS_CODES:
            raise ValueError(f"unknown formal solver {formal_solver!r}")
        d.formal_solver = _native.FS_CODES[formal_solver]
        d.gamma_per_ray = 1 if gamma_per_ray else 0
        d.layout = 1 if layout == "moments" else 0
        for name in ("t_nodes", "mu", "ang_w", "phi", "freq_w", "ybasis", "coeffs", "redistribution", "gamma",
                     "inflow"):
            if name in self._keep:
                setattr(d, name, dptr(self._keep[name]))
        h = ctypes.c_void_p()
        _native.check(lib.rtk_problem_create_slab(ctypes.byref(d), ctypes.byref(h)))
        self.h = h
        self.n_total = int(lib.rtk_problem_n_total(h))
        self.n_rays = n_angles * n_freq
        self._lib = lib

    def set_inflow(self, inflow: np.ndarray):
        arr = np.ascontiguousarray(inflow, dtype=float)
        _native.check(self._lib.rtk_problem_set_inflow(self.h, dptr(arr), arr.size, stream_ptr()))

    def set_tuning(self, key: str, value: int):
        """Select a kernel variant of this handle (rtk_problem_set_tuning); every variant
        computes the same operator."""
        _native.check(self._lib.rtk_problem_set_tuning(self.h, key.encode(), int(value)))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self._lib.rtk_problem_destroy(h)
            except Exception:  # pragma: no cover - interpreter shutdown
                pass
            self.h = None
