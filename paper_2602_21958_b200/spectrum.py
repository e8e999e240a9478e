"""Dense spectrum diagnostics of the global operator (R/spectrum.py).

The operator is materialised on the B200 (one device matvec per unit vector,
no host round trip per column; `operator.materialize_A`), then LAPACK's
nonsymmetric eigensolver runs on the host as in the reference.  Report fields
and cluster definitions follow R/spectrum.py:27-78: the symmetric modulus
interval [0.999, 1.001], the one-sided [0.999, 1] interval with a 1e-12 guard,
min |lambda| and outlier counts #{|lambda - 1| > eps}.
"""

from __future__ import annotations

import tempfile
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from paper_2602_21958_b200.errors import DENSE_CAP_DEFAULT
from paper_2602_21958_b200.operator import materialize_A

DEFAULT_EPS_VALUES = (0.01, 0.05, 0.1, 0.15)
_ONE_SIDED_GUARD = 1e-12


@dataclass
class SpectrumReport:
    eigenvalues: np.ndarray
    cluster_fraction: float            # symmetric: |lambda| in [0.999, 1.001]
    cluster_fraction_one_sided: float  # one-sided: |lambda| in [0.999, 1] (+ guard)
    min_modulus: float
    outlier_counts: dict               # eps -> #{|lambda - 1| > eps}
    descriptor: dict = field(default_factory=dict)
    singular_values: Optional[np.ndarray] = None

    @property
    def n(self) -> int:
        return self.eigenvalues.size


def spectrum_of(dense: np.ndarray, descriptor: dict = None, eps_values: Sequence[float] = DEFAULT_EPS_VALUES,
                compute_singular: bool = False) -> SpectrumReport:
    """Eigenvalues and cluster diagnostics of an already materialised operator."""
    try:
        eig = np.linalg.eigvals(dense)
    except np.linalg.LinAlgError as exc:   # pragma: no cover - LAPACK failure path
        path = tempfile.mktemp(prefix="rtk_b200_eig_fail_", suffix=".npy")
        np.save(path, dense)
        raise RuntimeError(f"eigensolver did not converge; matrix dumped to {path}") from exc
    modulus = np.abs(eig)
    distance = np.abs(eig - 1.0)
    desc = dict(descriptor or {})
    desc.update({"n_total": eig.size})
    return SpectrumReport(
        eigenvalues=eig,
        cluster_fraction=float(np.mean((modulus >= 0.999) & (modulus <= 1.001))),
        cluster_fraction_one_sided=float(np.mean((modulus >= 0.999) & (modulus <= 1.0 + _ONE_SIDED_GUARD))),
        min_modulus=float(modulus.min()),
        outlier_counts={float(e): int(np.sum(distance > e)) for e in eps_values},
        descriptor=desc,
        singular_values=np.linalg.svd(dense, compute_uv=False) if compute_singular else None,
    )


def compute_spectrum(problem, dense_cap: int = DENSE_CAP_DEFAULT, eps_values: Sequence[float] = DEFAULT_EPS_VALUES,
                     compute_singular: bool = False) -> SpectrumReport:
    """Full spectrum of the materialised operator plus diagnostics (R/spectrum.py:43-78)."""
    return spectrum_of(materialize_A(problem, dense_cap=dense_cap), problem.descriptor, eps_values,
                       compute_singular)


@dataclass
class TrendSummary:
    eps_values: tuple
    outlier_counts: dict
    cluster_fractions: list
    strong_cluster_consistent: bool


def clustering_trend(reports: Sequence[SpectrumReport], fluctuation: int = 2) -> TrendSummary:
    """Outlier-count trend along a refinement sequence (R/spectrum.py:89-117): consistent with a
    strong cluster when no count rises more than `fluctuation` above any earlier value."""
    if len(reports) < 2:
        raise ValueError("need at least two reports to assess a trend")
    eps_values = tuple(sorted(reports[0].outlier_counts))
    for rep in reports[1:]:
        if tuple(sorted(rep.outlier_counts)) != eps_values:
            raise ValueError("reports carry different eps grids")
    counts = {e: [rep.outlier_counts[e] for rep in reports] for e in eps_values}
    consistent = all(c <= min(series[:i + 1]) + fluctuation
                     for series in counts.values() for i, c in enumerate(series[1:]))
    return TrendSummary(eps_values=eps_values, outlier_counts=counts,
                        cluster_fractions=[rep.cluster_fraction for rep in reports],
                        strong_cluster_consistent=consistent)
