"""Partial-frequency-redistribution matrix R(nu, nu') (host-side setup).

The reference has no PRD kernel (R/scattering.py:52
is a closed Union of angle-only / coherent / CRD kernels).  This build fixes
the definition recorded in DESIGN.md:

    R0(x, x') = a * 1/2 erfc(max(|x|, |x'|)) + (1 - a) * phi(x) phi(x')

(Hummer's angle-averaged R_I, whose marginal is the normalised Gaussian
profile, mixed with complete redistribution), then scaled symmetrically,
R = D R0 D, so that the discrete quadrature conserves photons exactly:
    sum_f' R[f, f'] w_f' = phi_f.
Without that discrete normalisation GMRES(30) stalls.
"""

from __future__ import annotations

import math

import numpy as np


def gaussian_profile(x):
    """Doppler profile exp(-x^2)/sqrt(pi) in Doppler-width units."""
    x = np.asarray(x, dtype=float)
    return np.exp(-x * x) / math.sqrt(math.pi)


def prd_matrix(x, freq_w, phi, coherence: float = 0.5, tol: float = 1e-15, max_iter: int = 1000) -> np.ndarray:
    """Symmetric, discretely normalised PRD matrix on the frequency grid x."""
    x = np.asarray(x, dtype=float)
    w = np.asarray(freq_w, dtype=float)
    phi = np.asarray(phi, dtype=float)
    ax = np.abs(x)
    big = np.maximum.outer(ax, ax)
    erfc = np.frompyfunc(math.erfc, 1, 1)
    r0 = coherence * 0.5 * erfc(big).astype(float) + (1.0 - coherence) * np.outer(phi, phi)
    d = np.ones_like(x)
    for _ in range(max_iter):
        row = d * (r0 @ (d * w))
        if np.max(np.abs(row / phi - 1.0)) <= tol:
            break
        d = d * np.sqrt(phi / row)
    return d[:, None] * r0 * d[None, :]


def row_normalisation_error(R, freq_w, phi) -> float:
    """max_f |sum_f' R[f,f'] w_f' / phi_f - 1| (photon-conservation defect)."""
    return float(np.max(np.abs((np.asarray(R) @ np.asarray(freq_w)) / np.asarray(phi) - 1.0)))
