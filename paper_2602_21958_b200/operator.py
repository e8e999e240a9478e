"""Global operator A = I - Lambda Sigma on the B200 (R/operator.py).

`apply_A(problem, v)` keeps the reference signature (R/operator.py:48-53):
numpy in -> numpy out (one H2D, the fused device matvec, one D2H), or a torch
CUDA float64 tensor in -> tensor out with no copies.  The device problem
(tables + workspace) is uploaded once, on first use, and cached.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2602_21958_b200 import _device, _native
from paper_2602_21958_b200.errors import DENSE_CAP_DEFAULT, ResourceLimitError
from paper_2602_21958_b200.scattering import ScatteringOperator, slab_handle

__all__ = ["DENSE_CAP_DEFAULT", "ResourceLimitError", "RTProblem", "DeviceOperator", "apply_A", "apply_A_batch",
           "build_rhs",
           "source_function", "operator", "spectral_radius_estimate", "materialize_A",
           "intensity_from_moments"]


@dataclass
class RTProblem:
    """Grid, operators and thermal source of one setup (R/operator.py:28-45)."""

    grid: object
    transfer: object
    scattering: ScatteringOperator
    thermal: np.ndarray
    descriptor: dict = field(default_factory=dict)
    layout: str = "intensity"     # or "moments": unknown u = R_w M I, 2 N_nu N_s values
    _handle: object = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        self.thermal = np.asarray(self.thermal, dtype=float)
        if self.thermal.size == 1 and self.grid.n_total != 1:
            self.thermal = np.full(self.grid.n_total, float(self.thermal))
        if self.thermal.size != self.grid.n_total:
            raise ValueError("thermal source length does not match the grid")
        if self.layout not in ("intensity", "moments"):
            raise ValueError(f"unknown layout {self.layout!r}")

    @property
    def n_total(self) -> int:
        """Length of the unknown: the intensity vector, or the moment vector in the moment layout."""
        if self.layout == "moments":
            from paper_2602_21958_b200.scattering import separable_form

            return self.grid.n_space * separable_form(self.scattering.kernel, self.grid)[0].shape[0] * self.grid.n_freq
        return self.grid.n_total

    def device(self):
        """The uploaded device operator (built once)."""
        if self._handle is None:
            self._handle = slab_handle(self.grid, self.scattering, self.transfer, self.layout)
        return self._handle

    def invalidate(self):
        """Drop the device copy after editing grid/kernel/gamma/formal solver on the host."""
        self._handle = None


class DeviceOperator:
    """Callable v -> A v bound to a problem; lets gmres() run the fully native path."""

    def __init__(self, problem: RTProblem):
        self.problem = problem

    def __call__(self, v):
        return apply_A(self.problem, v)


def operator(problem: RTProblem) -> DeviceOperator:
    return DeviceOperator(problem)


def apply_A(problem: RTProblem, v):
    """v - Lambda(Sigma v), one fused device pass (R/operator.py:48-53)."""
    from paper_2602_21958_b200.lattice import LatticeProblem, lattice_apply_A

    if isinstance(problem, LatticeProblem):
        return lattice_apply_A(problem, v)
    n = problem.n_total
    h = problem.device()
    lib = _native.lib()
    if _device.is_tensor(v) and v.is_cuda:
        x, _ = _device.to_device(v, n)
        y = _device.empty(n)
        _native.check(lib.rtk_apply_A(h.h, _device.ptr(x), _device.ptr(y), n, _device.stream_ptr()))
        return y
    if _device.is_tensor(v):
        return apply_A(problem, v.cuda()).cpu()
    arr = np.ascontiguousarray(np.asarray(v, dtype=float).reshape(-1))
    if arr.size != n:
        raise ValueError(f"expected length {n}, got {arr.size}")
    out = np.empty(n)
    _native.check(lib.rtk_apply_A_host(h.h, _device.dptr(arr), _device.dptr(out), n, _device.stream_ptr()))
    return out


def apply_A_batch(problem: RTProblem, vs, out=None):
    """[A v for v in vs] for host (numpy) vectors, with the H2D copy of the next vector
    overlapping the D2H copy of the previous result (rtk_apply_A_host_batch).  Pass
    pinned-memory arrays (e.g. torch.empty(n, pin_memory=True).numpy()) for full overlap."""
    import ctypes

    n = problem.n_total
    h = problem.device()
    xs = [np.ascontiguousarray(np.asarray(v, dtype=float).reshape(-1)) for v in vs]
    for x in xs:
        if x.size != n:
            raise ValueError(f"expected length {n}, got {x.size}")
    ys = out if out is not None else [np.empty(n) for _ in xs]
    xp = (ctypes.c_void_p * len(xs))(*[x.ctypes.data for x in xs])
    yp = (ctypes.c_void_p * len(ys))(*[y.ctypes.data for y in ys])
    _native.check(_native.lib().rtk_apply_A_host_batch(h.h, xp, yp, len(xs), n))
    return ys


def build_rhs(problem: RTProblem, override_ones: bool = False, device: bool = False):
    """Lambda thermal + boundary term, or ones (R/operator.py:56-64)."""
    from paper_2602_21958_b200.lattice import LatticeProblem, lattice_build_rhs

    n = problem.n_total
    if isinstance(problem, LatticeProblem) and not override_ones:
        return lattice_build_rhs(problem, device=device)
    if override_ones:
        if device:
            torch = _device.require_cuda()
            return torch.ones(n, dtype=torch.float64, device="cuda")
        return np.ones(n)
    h = problem.device()
    h.set_inflow(problem.transfer.inflow)
    th, _ = _device.to_device(problem.thermal, problem.grid.n_total)
    b = _device.empty(n)
    _native.check(_native.lib().rtk_build_rhs(h.h, _device.ptr(th), _device.ptr(b), n, 0, _device.stream_ptr()))
    return b if device else b.cpu().numpy()


def intensity_from_moments(problem: RTProblem, u):
    """Moment layout: intensities I = Lambda(S(u) + thermal) + inflow term of a moment vector u."""
    if problem.layout != "moments":
        raise ValueError("intensity_from_moments needs a moment-layout problem")
    h = problem.device()
    h.set_inflow(problem.transfer.inflow)
    x, kind = _device.to_device(u, problem.n_total)
    ni = problem.grid.n_total
    th, _ = _device.to_device(problem.thermal, ni)
    out = _device.empty(ni)
    _native.check(_native.lib().rtk_intensity_from_moments(h.h, _device.ptr(x), _device.ptr(th), _device.ptr(out), ni,
                                                            _device.stream_ptr()))
    return _device.from_device(out, kind)


def source_function(problem: RTProblem, intensity):
    """S = Sigma I + thermal, the quantity the reference never exposes (R/operator.py:35)."""
    n = problem.n_total
    h = problem.device()
    x, kind = _device.to_device(intensity, n)
    th, _ = _device.to_device(problem.thermal, n)
    s = _device.empty(n)
    _native.check(_native.lib().rtk_source_function(h.h, _device.ptr(x), _device.ptr(th), _device.ptr(s), n,
                                                     _device.stream_ptr()))
    return _device.from_device(s, kind)


def spectral_radius_estimate(problem: RTProblem, iters: int = 50) -> float:
    """Power iteration on Lambda Sigma = I - A (R/operator.py:89-109), device vectors."""
    if iters < 1:
        raise ValueError("iters must be >= 1")
    torch = _device.require_cuda()
    rng = np.random.default_rng(12345)
    v = torch.from_numpy(rng.standard_normal(problem.n_total)).cuda()
    v /= torch.linalg.vector_norm(v)
    ratios = []
    for _ in range(iters):
        w = v - apply_A(problem, v)
        norm = float(torch.linalg.vector_norm(w))
        if norm == 0.0:
            return 0.0
        ratios.append(norm)
        v = w / norm
    tail = ratios[-min(5, len(ratios)):]
    return float(np.exp(np.mean(np.log(tail))))


def materialize_A(problem: RTProblem, dense_cap: int = DENSE_CAP_DEFAULT) -> np.ndarray:
    """Dense A by device matvecs on unit vectors (R/operator.py:67-86); tiny grids only."""
    n = problem.n_total
    if n > dense_cap:
        raise ResourceLimitError(f"dense operator of size {n} exceeds cap {dense_cap}")
    torch = _device.require_cuda()
    h = problem.device()
    lib = _native.lib()
    s = _device.stream_ptr()
    eye = torch.eye(n, dtype=torch.float64, device="cuda")      # row j = e_j
    cols = torch.empty((n, n), dtype=torch.float64, device="cuda")   # row j = A e_j
    row = 8 * n
    for j in range(n):   # stream-ordered, no host round trip per column
        _native.check(lib.rtk_apply_A(h.h, eye.data_ptr() + j * row, cols.data_ptr() + j * row, n, s))
    return cols.t().contiguous().cpu().numpy()
