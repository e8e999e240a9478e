"""B200-native (I - Lambda Sigma) operator and Krylov solvers for discrete-ordinates
radiative transfer -- a drop-in for the hot path of rtkrylov (arXiv 2602.21958).

The public names mirror the reference package (R/__init__.py:14-59) for the
hot path: grid / transfer / scattering setup on the host, then `apply_A`,
`build_rhs`, `gmres` / `bicgstab` / `solve_system` on the B200 through
librtk_b200.so (hand-written sm_100a kernels, C ABI in include/rtk_b200.h).
"""

__version__ = "0.1.0"

from paper_2602_21958_b200.errors import DENSE_CAP_DEFAULT, CoverageError, ResourceLimitError
from paper_2602_21958_b200.quadrature import QuadratureRule, gauss_legendre, legendre_basis, legendre_eval, trapezoid
from paper_2602_21958_b200.grid import (FieldVector, Grid, Ordering, Ray, build_grid, delta_tau, grid_from_nodes,
                                        permute)
from paper_2602_21958_b200.transfer import (TransferOperator, apply_transfer, boundary_term, build_transfer,
                                            materialize_transfer)
from paper_2602_21958_b200.scattering import (CoherentKernel, CRDKernel, DipolePRDKernel, LegendreKernel,
                                              ScatteringOperator, ScatteringStrengthWarning, apply_scattering,
                                              build_scattering, kernel_normalization, materialize_scattering,
                                              psi_matrix, separable_form)
from paper_2602_21958_b200.operator import (DeviceOperator, RTProblem, apply_A, apply_A_batch, build_rhs,
                                            intensity_from_moments, materialize_A, operator,
                                            source_function, spectral_radius_estimate)
from paper_2602_21958_b200.krylov import SolveConfig, SolveReport, bicgstab, gmres, solve_system
from paper_2602_21958_b200.redistribution import gaussian_profile, prd_matrix
from paper_2602_21958_b200.lattice import (LatticeProblem, dipole_harmonics, lattice_apply_A, lattice_build_rhs,
                                           lattice_problem, product_quadrature)
from paper_2602_21958_b200.spectrum import SpectrumReport, TrendSummary, clustering_trend, compute_spectrum
from paper_2602_21958_b200 import presets

__all__ = [
    "DENSE_CAP_DEFAULT", "CoverageError", "ResourceLimitError",
    "QuadratureRule", "gauss_legendre", "legendre_basis", "legendre_eval", "trapezoid",
    "FieldVector", "Grid", "Ordering", "Ray", "build_grid", "delta_tau", "grid_from_nodes", "permute",
    "TransferOperator", "apply_transfer", "boundary_term", "build_transfer", "materialize_transfer",
    "CoherentKernel", "CRDKernel", "DipolePRDKernel", "LegendreKernel", "ScatteringOperator",
    "ScatteringStrengthWarning", "apply_scattering", "build_scattering", "kernel_normalization",
    "materialize_scattering", "psi_matrix", "separable_form",
    "DeviceOperator", "RTProblem", "apply_A", "apply_A_batch", "build_rhs", "intensity_from_moments", "materialize_A", "operator", "source_function",
    "spectral_radius_estimate",
    "SolveConfig", "SolveReport", "bicgstab", "gmres", "solve_system",
    "SpectrumReport", "TrendSummary", "clustering_trend", "compute_spectrum", "presets",
    "gaussian_profile", "prd_matrix",
    "LatticeProblem", "dipole_harmonics", "lattice_apply_A", "lattice_build_rhs", "lattice_problem",
    "product_quadrature",
]
