"""Transfer operator Lambda (R/transfer.py), applied on the B200.

Block-diagonal per ray: downward rays (mu < 0) enter at the surface, upward
rays at depth (R/transfer.py:1-9).  `formal_solver` selects the reference's
implicit Euler ('ie', default, bit-compatible recursion) or the new
exponential integrators 'exp_linear' / 'exp_parabolic'.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from paper_2602_21958_b200 import _device, _native
from paper_2602_21958_b200.errors import DENSE_CAP_DEFAULT, ResourceLimitError
from paper_2602_21958_b200.grid import FieldVector, Grid, Ordering, permute

FORMAL_SOLVERS = ("ie", "exp_linear", "exp_parabolic")


def _per_frequency_values(grid: Grid, value) -> np.ndarray:
    """Boundary specification -> one value per ray (R/transfer.py:53-62)."""
    if callable(value):
        return np.asarray(value(grid.ray_nu), dtype=float) * np.ones(grid.n_rays)
    arr = np.asarray(value, dtype=float)
    if arr.ndim == 0:
        return np.full(grid.n_rays, float(arr))
    if arr.size == grid.n_freq:
        return np.tile(arr, grid.n_angles)
    raise ValueError(f"boundary values must be scalar or length {grid.n_freq}")


@dataclass
class TransferOperator:
    grid: Grid
    down: np.ndarray           # bool mask, rays entering at the surface
    inflow: np.ndarray         # (n_rays,) boundary intensity feeding each ray
    formal_solver: str = "ie"
    _handle: object = field(default=None, repr=False, compare=False)

    @property
    def n_total(self) -> int:
        return self.grid.n_total

    @property
    def dtau(self) -> np.ndarray:
        """(n_rays, n_space-1) increments (host view; the device recomputes them on the fly)."""
        return self.grid.delta_tau_table()

    def device(self):
        if self._handle is None:
            from paper_2602_21958_b200.scattering import slab_handle

            self._handle = slab_handle(self.grid, None, self)
        return self._handle

    # protocol shared with the multi-D operators (R/transfer.py:77-85)
    def apply_space_major(self, v):
        return apply_transfer(self, v)

    def boundary_space_major(self):
        return boundary_term(self).values

    def materialize(self, dense_cap: int = DENSE_CAP_DEFAULT) -> np.ndarray:
        return materialize_transfer(self, dense_cap)


def build_transfer(grid: Grid, i_in_deep=0.0, i_in_surf=0.0, formal_solver: str = "ie") -> TransferOperator:
    """Inflow per ray: deep value for mu > 0, surface value for mu < 0 (R/transfer.py:88-104)."""
    if formal_solver not in FORMAL_SOLVERS:
        raise ValueError(f"unknown formal solver {formal_solver!r}")
    down = grid.ray_mu < 0
    inflow = np.where(down, _per_frequency_values(grid, i_in_surf), _per_frequency_values(grid, i_in_deep))
    return TransferOperator(grid=grid, down=down, inflow=inflow, formal_solver=formal_solver)


def apply_transfer(op: TransferOperator, source):
    """Homogeneous part of Lambda on the device (R/transfer.py:134-141)."""
    is_fv = isinstance(source, FieldVector)
    ordering = source.ordering if is_fv else Ordering.SPACE_MAJOR
    vals = source.values if is_fv else source
    if is_fv and ordering is Ordering.RAY_MAJOR:
        vals = permute(op.grid, source, Ordering.SPACE_MAJOR).values
    h = op.device()
    x, kind = _device.to_device(vals, op.n_total)
    y = _device.empty(op.n_total)
    _native.check(_native.lib().rtk_apply_lambda(h.h, _device.ptr(x), _device.ptr(y), op.n_total,
                                                  _device.stream_ptr()))
    out = _device.from_device(y, kind)
    if not is_fv:
        return out
    fv = FieldVector(out, Ordering.SPACE_MAJOR)
    return permute(op.grid, fv, ordering) if ordering is Ordering.RAY_MAJOR else fv


def boundary_term(op: TransferOperator, device: bool = False) -> FieldVector:
    """Attenuated inflow, space-major (R/transfer.py:144-147), by an overflow-free recursion."""
    h = op.device()
    h.set_inflow(op.inflow)
    y = _device.empty(op.n_total)
    _native.check(_native.lib().rtk_boundary(h.h, _device.ptr(y), op.n_total, _device.stream_ptr()))
    return FieldVector(y if device else y.cpu().numpy(), Ordering.SPACE_MAJOR)


def materialize_transfer(op: TransferOperator, dense_cap: int = DENSE_CAP_DEFAULT) -> np.ndarray:
    """Dense Lambda by applying the device operator to unit vectors (R/transfer.py:150-161)."""
    n = op.n_total
    if n > dense_cap:
        raise ResourceLimitError(f"dense transfer of size {n} exceeds cap {dense_cap}")
    torch = _device.require_cuda()
    out = np.empty((n, n))
    e = torch.zeros(n, dtype=torch.float64, device="cuda")
    for j in range(n):
        e.zero_()
        e[j] = 1.0
        out[:, j] = apply_transfer(op, e).cpu().numpy()
    return out
