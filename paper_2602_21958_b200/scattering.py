"""Scattering operator Sigma = Gamma Psi W (R/scattering.py), applied on the B200.

Kernels keep the reference's types (LegendreKernel, CoherentKernel,
CRDKernel; R/scattering.py:28-52) and add DipolePRDKernel, the dipole
(l = 0 + 2) phase function times a partial-redistribution matrix R(nu, nu').
All of them reduce to one separable form
    Psi[(a,f),(a',f')] = sum_k c_k Y_k(a) Y_k(a') R[f,f'],
which is what the device kernels (moments -> R contraction -> on-the-fly
source expansion) evaluate.  Zero coefficients are dropped, so the dipole
kernel costs two moments, not three.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field
from typing import Callable, Union

import numpy as np

from paper_2602_21958_b200 import _device, _native
from paper_2602_21958_b200.errors import DENSE_CAP_DEFAULT, ResourceLimitError
from paper_2602_21958_b200.grid import FieldVector, Ordering, permute
from paper_2602_21958_b200.quadrature import legendre_basis


class ScatteringStrengthWarning(UserWarning):
    """Scattering strength outside the guaranteed fixed-point contraction regime."""


@dataclass(frozen=True)
class LegendreKernel:
    """sum_l d_l P_l(mu) P_l(mu'), frequency-flat (R/scattering.py:28-35)."""

    coefficients: tuple

    def __post_init__(self):
        object.__setattr__(self, "coefficients", tuple(float(c) for c in self.coefficients))


@dataclass(frozen=True)
class CoherentKernel:
    """Isotropic, no frequency redistribution (R/scattering.py:38-42)."""

    profile: Callable


@dataclass(frozen=True)
class CRDKernel:
    """Isotropic complete redistribution phi(nu) phi(nu') (R/scattering.py:45-49)."""

    profile: Callable


@dataclass(frozen=True, eq=False)
class DipolePRDKernel:
    """Dipole (Rayleigh-type) phase function x partial frequency redistribution.

    Psi = (sum_l d_l P_l(mu) P_l(mu')) (x) R(nu, nu') with d = (1, 0, 1/2),
    i.e. p = 1 + P_2(cos Theta)/2 azimuthally averaged.  `redistribution` is
    the (n_freq, n_freq) matrix on the grid's frequency nodes (see
    redistribution.prd_matrix).  New: the reference has no PRD kernel.
    """

    redistribution: np.ndarray
    coefficients: tuple = (1.0, 0.0, 0.5)

    def __post_init__(self):
        object.__setattr__(self, "coefficients", tuple(float(c) for c in self.coefficients))
        object.__setattr__(self, "redistribution", np.ascontiguousarray(self.redistribution, dtype=float))


Kernel = Union[LegendreKernel, CoherentKernel, CRDKernel, DipolePRDKernel]


def separable_form(kernel: Kernel, grid):
    """(ybasis (n_mom, n_angles), coeffs (n_mom,), R (n_freq, n_freq)) with zero rows dropped."""
    mu = np.asarray(grid.mu_nodes, dtype=float)
    nf = grid.n_freq
    if isinstance(kernel, (LegendreKernel, DipolePRDKernel)):
        d = np.asarray(kernel.coefficients, dtype=float)
        Y = legendre_basis(d.size - 1, mu)
        if isinstance(kernel, LegendreKernel):
            R = np.ones((nf, nf))
        else:
            R = kernel.redistribution
            if R.shape != (nf, nf):
                raise ValueError(f"redistribution must be ({nf}, {nf}), got {R.shape}")
        keep = d != 0.0
        if not np.any(keep):
            keep[0] = True
        Y, d = Y[keep], d[keep]
    elif isinstance(kernel, CRDKernel):
        pv = np.asarray(kernel.profile(grid.nu_nodes), dtype=float) * np.ones(nf)
        Y, d, R = np.ones((1, mu.size)), np.ones(1), np.outer(pv, pv)
    elif isinstance(kernel, CoherentKernel):
        pv = np.asarray(kernel.profile(grid.nu_nodes), dtype=float) * np.ones(nf)
        Y, d, R = np.ones((1, mu.size)), np.ones(1), np.diag(pv / grid.frequency_weights)
    else:
        raise TypeError(f"unknown kernel {kernel!r}")
    if d.size > _native.MAX_MOMENTS:
        raise ValueError(f"at most {_native.MAX_MOMENTS} nonzero kernel moments are supported")
    return np.ascontiguousarray(Y), np.ascontiguousarray(d), np.ascontiguousarray(R, dtype=float)


def psi_matrix(kernel: Kernel, grid) -> np.ndarray:
    """Dense kernel matrix over ray pairs (R/scattering.py:55-71); host helper for tiny grids."""
    Y, d, R = separable_form(kernel, grid)
    ang = Y.T @ (d[:, None] * Y)
    ang = np.triu(ang) + np.triu(ang, 1).T
    return np.kron(ang, R)


def kernel_normalization(kernel: Kernel, grid) -> float:
    """w^T Psi w / sphere_measure^2 (R/scattering.py:162-175), evaluated in separable form."""
    Y, d, R = separable_form(kernel, grid)
    wa = np.asarray(grid.angular_weights, dtype=float)
    wf = np.asarray(grid.frequency_weights, dtype=float)
    ang = float(np.sum(d * (Y @ wa) ** 2))
    return ang * float(wf @ (R @ wf)) / grid.sphere_measure ** 2


def split_gamma(gamma_table: np.ndarray, grid):
    """(gamma, per_ray): (n_space, n_freq) when gamma does not depend on mu
    (every reference preset and BASELINE config), else the full table."""
    g = np.asarray(gamma_table, dtype=float).reshape(grid.n_space, grid.n_angles, grid.n_freq)
    if np.all(g == g[:, :1, :]):
        return np.ascontiguousarray(g[:, 0, :]), False
    return np.ascontiguousarray(gamma_table, dtype=float), True


@dataclass
class ScatteringOperator:
    grid: object
    kernel: Kernel
    gamma_table: np.ndarray  # (n_space, n_rays), the reference's layout
    _handle: object = field(default=None, repr=False, compare=False)

    @property
    def n_total(self) -> int:
        return self.grid.n_total

    def device(self):
        if self._handle is None:
            self._handle = slab_handle(self.grid, self, None)
        return self._handle


def slab_handle(grid, scattering, transfer, layout: str = "intensity"):
    """Upload one slab problem; scattering or transfer may be None (identity-free stand-ins)."""
    if scattering is not None:
        Y, d, R = separable_form(scattering.kernel, grid)
        gamma, per_ray = split_gamma(scattering.gamma_table, grid)
    else:
        Y, d, R = np.ones((1, grid.n_angles)), np.zeros(1), np.zeros((grid.n_freq, grid.n_freq))
        gamma, per_ray = np.zeros((grid.n_space, grid.n_freq)), False
    fs = transfer.formal_solver if transfer is not None else "ie"
    inflow = transfer.inflow if transfer is not None else None
    arrays = dict(t_nodes=grid.t_nodes, mu=grid.mu_nodes, ang_w=grid.angular_weights, phi=grid.profile_values(),
                  freq_w=grid.frequency_weights, ybasis=Y, coeffs=d, redistribution=R, gamma=gamma, inflow=inflow)
    return _device.SlabHandle(arrays, fs, per_ray, grid.n_space, grid.n_angles, grid.n_freq, Y.shape[0], layout)


def build_scattering(grid, kernel: Kernel, gamma) -> ScatteringOperator:
    """Sample gamma on the node x ray grid; warn when the strength reaches one (R/scattering.py:85-100)."""
    gamma_table = grid.sample_coefficient(gamma)
    strength = float(np.max(np.abs(gamma_table))) * kernel_normalization(kernel, grid)
    if strength >= 1.0:
        warnings.warn(f"scattering strength {strength:.3g} >= 1: fixed-point iteration may not contract "
                      "(Krylov solvers are unaffected)", ScatteringStrengthWarning, stacklevel=2)
    return ScatteringOperator(grid=grid, kernel=kernel, gamma_table=gamma_table)


def _unwrap(op, v):
    if isinstance(v, FieldVector):
        vals = v.values
        if v.ordering is Ordering.RAY_MAJOR:
            vals = permute(op.grid, v, Ordering.SPACE_MAJOR).values
        return vals, v.ordering, True
    return v, Ordering.SPACE_MAJOR, False


def _wrap(op, out, ordering, is_fv):
    if not is_fv:
        return out
    fv = FieldVector(out, Ordering.SPACE_MAJOR)
    return permute(op.grid, fv, ordering) if ordering is Ordering.RAY_MAJOR else fv


def apply_scattering(op: ScatteringOperator, field_) -> object:
    """Matrix-free Gamma Psi W on the device (R/scattering.py:126-148)."""
    vals, ordering, is_fv = _unwrap(op, field_)
    h = op.device()
    x, kind = _device.to_device(vals, op.n_total)
    y = _device.empty(op.n_total)
    _native.check(_native.lib().rtk_apply_sigma(h.h, _device.ptr(x), _device.ptr(y), op.n_total,
                                                 _device.stream_ptr()))
    return _wrap(op, _device.from_device(y, kind), ordering, is_fv)


def materialize_scattering(op: ScatteringOperator, dense_cap: int = DENSE_CAP_DEFAULT) -> np.ndarray:
    """Dense Gamma Psi W (R/scattering.py:151-159), host helper for tiny grids."""
    n = op.n_total
    if n > dense_cap:
        raise ResourceLimitError(f"dense scattering of size {n} exceeds cap {dense_cap}")
    g = op.grid
    psi_w = psi_matrix(op.kernel, g) * g.combined_weights[None, :]
    out = np.zeros((n, n))
    view = out.reshape(g.n_space, g.n_rays, g.n_space, g.n_rays)
    for i in range(g.n_space):
        view[i, :, i, :] = op.gamma_table[i][:, None] * psi_w
    return out
