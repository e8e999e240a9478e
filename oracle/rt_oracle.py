"""numpy restatement of the rtkrylov hot path (TEST INFRASTRUCTURE, see oracle/__init__.py).

Every function cites the reference file:line it restates.  R/ is
/root/reference/pkg/src/rtkrylov/.  Functions marked EXTENSION have no
reference implementation (the BASELINE configs need them); their pinning is
described in DESIGN.md "Parity".

The oracle works on plain arrays ("descriptions"), so the same setup arrays
can be fed to the B200 build and to this checker.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

__all__ = [
    "gauss_legendre", "trapezoid", "legendre_basis", "gaussian_profile",
    "SlabDesc", "slab_desc", "delta_tau_table",
    "sweep_down", "sweep_up", "exp_weights", "EXP_SERIES_THRESHOLD",
    "apply_transfer", "boundary_term", "apply_sigma", "apply_A", "build_rhs",
    "materialize", "psi_dipole_prd", "prd_matrix", "legendre_as_general",
    "crd_as_general", "coherent_as_general", "OracleSolveReport", "gmres",
    "bicgstab", "source_function", "desc_from_problem", "moments_of", "source_from_moments",
    "apply_A_moments", "build_rhs_moments", "intensity_from_moments",
]


# ---------------------------------------------------------------------------
# quadrature (R/quadrature.py)
# ---------------------------------------------------------------------------

def legendre_basis(l_max: int, x) -> np.ndarray:
    """P_0..P_lmax at x, Bonnet recurrence in the reference's order (R/quadrature.py:49-58)."""
    x = np.asarray(x, dtype=float)
    out = np.empty((l_max + 1, x.size))
    out[0] = 1.0
    if l_max >= 1:
        out[1] = x
    for k in range(1, l_max):
        out[k + 1] = ((2 * k + 1) * x * out[k] - k * out[k - 1]) / (k + 1)
    return out


def _p_and_dp(n, x):
    # R/quadrature.py:61-67
    p_prev = np.ones_like(x)
    p = x.copy()
    for k in range(1, n):
        p, p_prev = ((2 * k + 1) * x * p - k * p_prev) / (k + 1), p
    dp = n * (x * p - p_prev) / (x * x - 1.0)
    return p, dp


def gauss_legendre(n: int, lo: float = -1.0, hi: float = 1.0):
    """Newton on P_n from Chebyshev guesses, tol 1e-15, 100 iterations (R/quadrature.py:70-100)."""
    if n < 1 or not lo < hi:
        raise ValueError("bad Gauss-Legendre request")
    if n == 1:
        x = np.array([0.0])
        w = np.array([2.0])
    else:
        i = np.arange(n)
        x = np.cos(np.pi * (4 * i + 3) / (4 * n + 2))
        for _ in range(100):
            p, dp = _p_and_dp(n, x)
            dx = p / dp
            x -= dx
            if np.max(np.abs(dx)) < 1e-15:
                break
        _, dp = _p_and_dp(n, x)
        w = 2.0 / ((1.0 - x * x) * dp * dp)
        order = np.argsort(x)
        x, w = x[order], w[order]
    half = 0.5 * (hi - lo)
    return 0.5 * (lo + hi) + half * x, half * w


def trapezoid(n: int, lo: float, hi: float):
    """Composite trapezoid rule including endpoints (R/quadrature.py:103-113)."""
    if n < 2 or not lo < hi:
        raise ValueError("bad trapezoid request")
    nodes = np.linspace(lo, hi, n)
    h = (hi - lo) / (n - 1)
    w = np.full(n, h)
    w[0] = w[-1] = 0.5 * h
    return nodes, w


def gaussian_profile(x):
    """EXTENSION (BASELINE configs): Doppler profile exp(-x^2)/sqrt(pi)."""
    x = np.asarray(x, dtype=float)
    return np.exp(-x * x) / math.sqrt(math.pi)


# ---------------------------------------------------------------------------
# 1D slab description (R/grid.py:63-112, R/transfer.py:88-104, R/scattering.py:85-100)
# ---------------------------------------------------------------------------

@dataclass
class SlabDesc:
    """Everything the 1D matvec needs, as plain arrays.

    Ray order is direction-major, frequency-minor and the flat vector is
    space-major: index = i * n_rays + a * n_freq + f (R/grid.py:83-88).
    Sigma is the general separable kernel
        Psi[(a,f),(a',f')] = sum_k coeffs[k] Y[k,a] Y[k,a'] * R[f,f']
    which covers LegendreKernel (Y = P_l, R = ones), CRDKernel (Y = 1,
    R = phi phi'), CoherentKernel (Y = 1, R = diag(phi / w_f)) and the
    EXTENSION dipole x PRD kernel (Y = P_0, P_2, coeffs = (1, 1/2)).
    """

    t_nodes: np.ndarray
    mu: np.ndarray
    ang_w: np.ndarray
    nu: np.ndarray
    freq_w: np.ndarray
    phi: np.ndarray                 # profile at nu nodes
    ybasis: np.ndarray              # (n_mom, n_angles)
    coeffs: np.ndarray              # (n_mom,)
    R: np.ndarray                   # (n_freq, n_freq)
    gamma: np.ndarray               # (n_space, n_rays) -- reference gamma_table layout
    thermal: np.ndarray             # (n_total,)
    inflow: np.ndarray              # (n_rays,) surface value for mu<0 rays, deep value for mu>0
    formal_solver: str = "ie"

    @property
    def n_space(self):
        return self.t_nodes.size

    @property
    def n_angles(self):
        return self.mu.size

    @property
    def n_freq(self):
        return self.nu.size

    @property
    def n_rays(self):
        return self.n_angles * self.n_freq

    @property
    def n_total(self):
        return self.n_space * self.n_rays

    @property
    def ray_mu(self):
        return np.repeat(self.mu, self.n_freq)

    @property
    def down(self):
        return self.ray_mu < 0


def delta_tau_table(d: SlabDesc) -> np.ndarray:
    """phi(nu) * dt / |mu| per ray, evaluated in the reference's order (R/grid.py:101-105)."""
    dt = np.diff(d.t_nodes)
    phi_r = np.tile(d.phi, d.n_angles)
    return phi_r[:, None] * dt[None, :] / np.abs(d.ray_mu)[:, None]


def slab_desc(t_nodes, n_angles, nu, freq_w, phi, ybasis_fn, coeffs, R, gamma_fn,
              thermal=0.0, i_in_deep=0.0, i_in_surf=0.0, formal_solver="ie") -> SlabDesc:
    """Assemble a description the way build_grid/build_transfer/build_scattering do
    (R/grid.py:137-140 half-interval GL; R/transfer.py:101-103 inflow; R/grid.py:107-112 gamma)."""
    t_nodes = np.asarray(t_nodes, dtype=float)
    dn_x, dn_w = gauss_legendre(n_angles // 2, -1.0, 0.0)
    up_x, up_w = gauss_legendre(n_angles // 2, 0.0, 1.0)
    mu = np.concatenate([dn_x, up_x])
    ang_w = np.concatenate([dn_w, up_w])
    nu = np.asarray(nu, dtype=float)
    n_f = nu.size
    ray_mu = np.repeat(mu, n_f)
    ray_nu = np.tile(nu, mu.size)
    gamma = np.ascontiguousarray(np.broadcast_to(
        np.asarray(gamma_fn(t_nodes[:, None], ray_mu[None, :], ray_nu[None, :]), dtype=float),
        (t_nodes.size, ray_mu.size)))
    n_total = t_nodes.size * ray_mu.size
    th = np.asarray(thermal, dtype=float)
    th = np.full(n_total, float(th)) if th.ndim == 0 else th.reshape(n_total)
    deep = np.broadcast_to(np.asarray(i_in_deep, dtype=float), (n_f,)) if np.ndim(i_in_deep) else np.full(n_f, float(i_in_deep))
    surf = np.broadcast_to(np.asarray(i_in_surf, dtype=float), (n_f,)) if np.ndim(i_in_surf) else np.full(n_f, float(i_in_surf))
    inflow = np.where(ray_mu < 0, np.tile(surf, mu.size), np.tile(deep, mu.size))
    return SlabDesc(t_nodes=t_nodes, mu=mu, ang_w=ang_w, nu=nu, freq_w=np.asarray(freq_w, dtype=float),
                    phi=np.asarray(phi, dtype=float), ybasis=np.asarray(ybasis_fn(mu), dtype=float),
                    coeffs=np.asarray(coeffs, dtype=float), R=np.asarray(R, dtype=float),
                    gamma=gamma, thermal=th, inflow=inflow, formal_solver=formal_solver)


# ---------------------------------------------------------------------------
# kernels expressed in the general separable form
# ---------------------------------------------------------------------------

def legendre_as_general(coefficients, mu, n_freq):
    """LegendreKernel (R/scattering.py:28-35, apply at 132-136): Y = P_l(mu), R = ones."""
    d = np.asarray(coefficients, dtype=float)
    return legendre_basis(d.size - 1, mu), d, np.ones((n_freq, n_freq))


def crd_as_general(phi, mu):
    """CRDKernel (R/scattering.py:45-49, apply at 137-140): Y = 1, R = phi phi^T."""
    return np.ones((1, mu.size)), np.ones(1), np.outer(phi, phi)


def coherent_as_general(phi, freq_w, mu):
    """CoherentKernel (R/scattering.py:38-42, psi at 65-70, apply at 141-145): R = diag(phi / w_f)."""
    return np.ones((1, mu.size)), np.ones(1), np.diag(np.asarray(phi) / np.asarray(freq_w))


def prd_matrix(x, freq_w, phi, a: float = 0.5, tol: float = 1e-15, max_iter: int = 1000):
    """EXTENSION: partial-redistribution matrix R(nu, nu').

    R0 = a * 1/2 erfc(max(|x|, |x'|)) + (1 - a) phi(x) phi(x'): Hummer's
    angle-averaged R_I (marginal phi) mixed with complete redistribution.
    Symmetric Sinkhorn scaling R = D R0 D makes the discrete quadrature
    exact: sum_f' R[f, f'] w_f' = phi_f (photon conservation on the grid).
    """
    x = np.asarray(x, dtype=float)
    ax = np.abs(x)
    big = np.maximum(ax[:, None], ax[None, :])
    erfc = np.vectorize(math.erfc)
    R0 = a * 0.5 * erfc(big) + (1.0 - a) * np.outer(phi, phi)
    d = np.ones_like(x)
    w = np.asarray(freq_w, dtype=float)
    phi = np.asarray(phi, dtype=float)
    for _ in range(max_iter):
        r = d * (R0 @ (d * w))
        err = np.max(np.abs(r / phi - 1.0))
        if err <= tol:
            break
        d = d * np.sqrt(phi / r)
    return d[:, None] * R0 * d[None, :]


def psi_dipole_prd(ybasis, coeffs, R):
    """Dense Psi = sum_k c_k Y_k Y_k^T  (x)  R over the ray order (cf. psi_matrix, R/scattering.py:55-71)."""
    ang = ybasis.T @ (np.asarray(coeffs)[:, None] * ybasis)
    return np.kron(ang, R)


# ---------------------------------------------------------------------------
# formal solvers: sweeps over (n_rays, n_space) blocks
# ---------------------------------------------------------------------------

EXP_SERIES_THRESHOLD = 0.05
# h1(d) = e1/d^2 = sum_{n=2}^{9} (-1)^n d^(n-2)/n!;  h2(d) = e2/d^3 = 2 sum_{n=3}^{10} (-1)^(n+1) d^(n-3)/n!
_H1 = [((-1) ** n) / math.factorial(n) for n in range(2, 10)]
_H2 = [2.0 * ((-1) ** (n + 1)) / math.factorial(n) for n in range(3, 11)]


def _horner(coefs, d):
    acc = np.zeros_like(d) + coefs[-1]
    for c in coefs[-2::-1]:
        acc = acc * d + c
    return acc


def exp_weights(d):
    """EXTENSION: (att = e^-d, e0, e1, e2) with e_k = int_0^d t^k e^{-(d - t)} dt.

    Shared with the CUDA build (csrc/formal.cuh) and the C port:
      d < 0.05 : e1 = d^2 h1(d), e2 = d^3 h2(d) (8-term Taylor series), e0 = d - e1, att = 1 - e0;
      else     : att = exp(-d), e0 = 1 - att, e1 = d - e0, e2 = d^2 - 2 e1.
    """
    d = np.asarray(d, dtype=float)
    small = d < EXP_SERIES_THRESHOLD
    with np.errstate(over="ignore", invalid="ignore"):
        att_big = np.exp(-d)
        e1_small = d * d * _horner(_H1, d)
        e2_small = d * d * d * _horner(_H2, d)
    e0 = np.where(small, d - e1_small, 1.0 - att_big)
    att = np.where(small, 1.0 - e0, att_big)
    e1 = np.where(small, e1_small, d - e0)
    e2 = np.where(small, e2_small, d * d - 2.0 * e1)
    return att, e0, e1, e2


def _linear_weights(d):
    """(att, w_u, w_c) as csrc/formal.cuh: series path w_c = d h1(d), e0 = d - d w_c, att = 1 - e0;
    transcendental path att = exp(-d), e0 = 1 - att, w_c = (d - e0) / d."""
    d = np.asarray(d, dtype=float)
    small = d < EXP_SERIES_THRESHOLD
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        wc_s = d * _horner(_H1, d)
        att_b = np.exp(-d)
        e0_b = 1.0 - att_b
        wc_b = (d - e0_b) / d
    e0 = np.where(small, d - d * wc_s, e0_b)
    att = np.where(small, 1.0 - e0, att_b)
    wc = np.where(small, wc_s, wc_b)
    return att, e0 - wc, wc


def _parabolic_weights(du, dd):
    att, e0, e1, e2 = exp_weights(du)
    s = du + dd
    r = 1.0 / (du * dd * s)          # one division shared by the three weights (csrc/formal.cuh)
    wu = e0 + (e2 - (dd + 2.0 * du) * e1) * (dd * r)
    wc = (s * e1 - e2) * (s * r)
    wd = (e2 - du * e1) * (du * r)
    return att, wu, wc, wd


def sweep_down(dtau, src, acc0=None, solver="ie"):
    """Downward march entering at node 0 (R/_kernels.py:37-45 for IE).

    IE: out_{i+1} = (out_i + dtau_i src_{i+1}) / (1 + dtau_i), the reference's
    division form.  acc0 (default 0) is the inflow value carried by node 0,
    which makes the same recursion produce the boundary term without the
    reference's cumprod overflow (SURVEY.md section 5 defect 1).
    EXTENSION solvers: 'exp_linear' (Olson-Kunasz), 'exp_parabolic'
    (Kunasz-Auer; linear on the last segment).
    """
    dtau = np.asarray(dtau, dtype=float)
    src = np.asarray(src, dtype=float)
    m, n = src.shape
    out = np.empty_like(src)
    acc = np.zeros(m) if acc0 is None else np.array(acc0, dtype=float).reshape(m)
    out[:, 0] = acc
    for i in range(n - 1):
        d = dtau[:, i]
        if solver == "ie":
            acc = (acc + d * src[:, i + 1]) / (1.0 + d)
        elif solver == "exp_linear" or (solver == "exp_parabolic" and i == n - 2):
            att, wu, wc = _linear_weights(d)
            acc = att * acc + wu * src[:, i] + wc * src[:, i + 1]
        elif solver == "exp_parabolic":
            att, wu, wc, wd = _parabolic_weights(d, dtau[:, i + 1])
            acc = att * acc + wu * src[:, i] + wc * src[:, i + 1] + wd * src[:, i + 2]
        else:
            raise ValueError(f"unknown formal solver {solver!r}")
        out[:, i + 1] = acc
    return out


def sweep_up(dtau, src, acc0=None, solver="ie"):
    """Upward march entering at node n-1 (R/_kernels.py:48-54 for IE):
    out_{i-1} = (out_i + dtau_{i-1} src_{i-1}) / (1 + dtau_{i-1})."""
    rev = sweep_down(np.asarray(dtau)[:, ::-1], np.asarray(src)[:, ::-1], acc0, solver)
    return rev[:, ::-1]


def apply_transfer(d: SlabDesc, source: np.ndarray, with_boundary: bool = False) -> np.ndarray:
    """Homogeneous Lambda on a space-major vector (R/transfer.py:134-141)."""
    mat = np.ascontiguousarray(np.asarray(source, dtype=float).reshape(d.n_space, d.n_rays).T)
    dtau = delta_tau_table(d)
    down = d.down
    up = ~down
    out = np.empty_like(mat)
    acc_dn = d.inflow[down] if with_boundary else None
    acc_up = d.inflow[up] if with_boundary else None
    out[down] = sweep_down(dtau[down], mat[down], acc_dn, d.formal_solver)
    out[up] = sweep_up(dtau[up], mat[up], acc_up, d.formal_solver)
    return out.T.ravel()


def boundary_term(d: SlabDesc) -> np.ndarray:
    """decay * inflow (R/transfer.py:144-147), computed as a zero-source sweep
    from the inflow value so it cannot overflow (R/transfer.py:97-99 does)."""
    return apply_transfer(d, np.zeros(d.n_total), with_boundary=True)


def apply_sigma(d: SlabDesc, field_: np.ndarray) -> np.ndarray:
    """Matrix-free Gamma Psi W per space node in moment form (R/scattering.py:126-148):
        m[i,k,f'] = sum_a w_a Y_k(a) I[i,a,f']
        M[i,k,f]  = sum_f' R[f,f'] w_f' m[i,k,f']
        S[i,a,f]  = gamma[i,(a,f)] sum_k c_k Y_k(a) M[i,k,f]
    """
    cube = np.asarray(field_, dtype=float).reshape(d.n_space, d.n_angles, d.n_freq)
    m = np.einsum("saf,ka->skf", cube, d.ybasis * d.ang_w[None, :])
    M = np.einsum("fg,skg->skf", d.R * d.freq_w[None, :], m)
    S = np.einsum("ka,skf->saf", d.coeffs[:, None] * d.ybasis, M)
    return (d.gamma * S.reshape(d.n_space, d.n_rays)).ravel()


def apply_A(d: SlabDesc, v: np.ndarray) -> np.ndarray:
    """v - Lambda(Sigma v) (R/operator.py:48-53)."""
    v = np.asarray(v, dtype=float)
    if v.size != d.n_total:
        raise ValueError(f"expected length {d.n_total}, got {v.size}")
    return v - apply_transfer(d, apply_sigma(d, v))


def build_rhs(d: SlabDesc, override_ones: bool = False) -> np.ndarray:
    """Lambda thermal + boundary term (R/operator.py:56-64)."""
    if override_ones:
        return np.ones(d.n_total)
    return apply_transfer(d, d.thermal) + boundary_term(d)


def moments_of(d: SlabDesc, I: np.ndarray) -> np.ndarray:
    """EXTENSION (moment layout): u = R_w M I, u[i,k,f] = sum_g R[f,g] w_g sum_a w_a Y_k(a) I[i,a,g]."""
    cube = np.asarray(I, dtype=float).reshape(d.n_space, d.n_angles, d.n_freq)
    m = np.einsum("saf,ka->skf", cube, d.ybasis * d.ang_w[None, :])
    return np.einsum("fg,skg->skf", d.R * d.freq_w[None, :], m).reshape(-1)


def source_from_moments(d: SlabDesc, u: np.ndarray) -> np.ndarray:
    """S[i,a,f] = gamma[i,(a,f)] sum_k c_k Y_k(a) u[i,k,f]."""
    u3 = np.asarray(u, dtype=float).reshape(d.n_space, d.ybasis.shape[0], d.n_freq)
    S = np.einsum("ka,skf->saf", d.coeffs[:, None] * d.ybasis, u3)
    return (d.gamma * S.reshape(d.n_space, d.n_rays)).ravel()


def apply_A_moments(d: SlabDesc, u: np.ndarray) -> np.ndarray:
    """EXTENSION: y = u - R_w M Lambda S(u), the operator in moment coordinates."""
    return np.asarray(u, dtype=float) - moments_of(d, apply_transfer(d, source_from_moments(d, u)))


def build_rhs_moments(d: SlabDesc) -> np.ndarray:
    return moments_of(d, build_rhs(d))


def intensity_from_moments(d: SlabDesc, u: np.ndarray) -> np.ndarray:
    """I = Lambda(S(u) + thermal) + inflow term."""
    return apply_transfer(d, source_from_moments(d, u) + d.thermal, with_boundary=True)


def source_function(d: SlabDesc, intensity: np.ndarray) -> np.ndarray:
    """S = Sigma I + thermal (R/scattering.py:126 + R/operator.py:35; no reference helper)."""
    return apply_sigma(d, intensity) + d.thermal


def desc_from_problem(problem) -> SlabDesc:
    """Oracle description of a product-side (paper_2602_21958_b200) RTProblem, read by duck
    typing: the same setup arrays, with the kernel mapped by this module's own restatement
    (legendre_as_general / crd_as_general / coherent_as_general), not by product code."""
    g = problem.grid
    k = problem.scattering.kernel
    kind = type(k).__name__
    phi = np.asarray(g.profile(g.nu_nodes), dtype=float) * np.ones(g.n_freq)
    if kind in ("LegendreKernel", "DipolePRDKernel"):
        Y, c, R = legendre_as_general(k.coefficients, g.mu_nodes, g.n_freq)
        if kind == "DipolePRDKernel":
            R = np.asarray(k.redistribution, dtype=float)
        keep = c != 0.0
        Y, c = Y[keep], c[keep]
    elif kind == "CRDKernel":
        Y, c, R = crd_as_general(np.asarray(k.profile(g.nu_nodes), dtype=float) * np.ones(g.n_freq), g.mu_nodes)
    elif kind == "CoherentKernel":
        Y, c, R = coherent_as_general(np.asarray(k.profile(g.nu_nodes), dtype=float) * np.ones(g.n_freq),
                                      g.frequency_weights, g.mu_nodes)
    else:
        raise TypeError(kind)
    return SlabDesc(t_nodes=g.t_nodes, mu=g.mu_nodes, ang_w=g.angular_weights, nu=g.nu_nodes,
                    freq_w=g.frequency_weights, phi=phi, ybasis=Y, coeffs=c, R=R,
                    gamma=np.asarray(problem.scattering.gamma_table, dtype=float),
                    thermal=np.asarray(problem.thermal, dtype=float),
                    inflow=np.asarray(problem.transfer.inflow, dtype=float),
                    formal_solver=problem.transfer.formal_solver)


def materialize(apply: Callable[[np.ndarray], np.ndarray], n: int) -> np.ndarray:
    """Dense matrix by applying to unit vectors (oracle for tiny n)."""
    out = np.empty((n, n))
    e = np.zeros(n)
    for j in range(n):
        e[j] = 1.0
        out[:, j] = apply(e)
        e[j] = 0.0
    return out


# ---------------------------------------------------------------------------
# Krylov (R/krylov.py)
# ---------------------------------------------------------------------------

@dataclass
class OracleSolveReport:
    solution: np.ndarray
    iterations: int
    residual_history: list
    converged: bool
    method: str
    breakdown: bool = False
    true_residual: Optional[float] = None
    residual_kind: str = "recurrence"


def gmres(apply, b, rel_tol=1e-12, max_iter=1000, restart=None, reorthogonalize=False):
    """Restarted GMRES, MGS Arnoldi, Givens least squares, x0 = 0, breakdown at
    1e-14 ||b||, true-residual guard at 10 tol (R/krylov.py:56-158, 161-177)."""
    b = np.asarray(b, dtype=float)
    n = b.size
    b_norm = float(np.linalg.norm(b))
    if b_norm == 0.0:
        return OracleSolveReport(np.zeros(n), 0, [0.0], True, "gmres", true_residual=0.0)
    history = []
    x = np.zeros(n)
    r = b.copy()
    total = 0
    cycle = restart if restart is not None else max_iter
    while total < max_iter:
        beta = float(np.linalg.norm(r))
        if beta / b_norm <= rel_tol:
            history.append(beta / b_norm)
            return OracleSolveReport(x, max(total, 1), history, True, "gmres", true_residual=beta / b_norm)
        basis = [r / beta]
        h_cols, cos, sin, g = [], [], [], [beta]
        breakdown = False
        steps = min(cycle, max_iter - total)
        j = 0
        while j < steps:
            w = np.array(apply(basis[j]), dtype=float)
            col = np.empty(j + 2)
            for i in range(j + 1):
                col[i] = float(np.dot(basis[i], w))
                w -= col[i] * basis[i]
            if reorthogonalize:
                for i in range(j + 1):
                    c = float(np.dot(basis[i], w))
                    col[i] += c
                    w -= c * basis[i]
            col[j + 1] = float(np.linalg.norm(w))
            breakdown = col[j + 1] < 1e-14 * b_norm
            if not breakdown:
                basis.append(w / col[j + 1])
            for i in range(j):
                tmp = cos[i] * col[i] + sin[i] * col[i + 1]
                col[i + 1] = -sin[i] * col[i] + cos[i] * col[i + 1]
                col[i] = tmp
            denom = np.hypot(col[j], col[j + 1])
            cj = col[j] / denom if denom else 1.0
            sj = col[j + 1] / denom if denom else 0.0
            cos.append(cj)
            sin.append(sj)
            col[j] = denom
            h_cols.append(col[: j + 1].copy())
            g.append(-sj * g[j])
            g[j] = cj * g[j]
            total += 1
            j += 1
            rel = abs(g[j]) / b_norm
            history.append(rel)
            if rel <= rel_tol or breakdown:
                y = _solve_upper(h_cols, g[:j])
                cand = x + _combine(basis, y)
                true_rel = float(np.linalg.norm(b - apply(cand))) / b_norm
                if true_rel <= 10.0 * rel_tol:
                    if breakdown:
                        history[-1] = true_rel
                    return OracleSolveReport(cand, total, history, True, "gmres", breakdown, true_rel)
                if breakdown:
                    return OracleSolveReport(cand, total, history, False, "gmres", True, true_rel)
        y = _solve_upper(h_cols, g[:j])
        x = x + _combine(basis, y)
        r = b - apply(x)
    return OracleSolveReport(x, total, history, False, "gmres",
                             true_residual=float(np.linalg.norm(r)) / b_norm)


def _solve_upper(h_cols, g):
    # R/krylov.py:161-170
    m = len(g)
    y = np.zeros(m)
    for i in range(m - 1, -1, -1):
        s = g[i]
        for k in range(i + 1, m):
            s -= h_cols[k][i] * y[k]
        y[i] = s / h_cols[i][i]
    return y


def _combine(basis, y):
    # R/krylov.py:173-177
    out = y[0] * basis[0]
    for i in range(1, y.size):
        out = out + y[i] * basis[i]
    return out


def bicgstab(apply, b, rel_tol=1e-12, max_iter=1000):
    """BiCGStab with shadow residual r0, breakdown at 1e-30 (R/krylov.py:180-256)."""
    b = np.asarray(b, dtype=float)
    n = b.size
    b_norm = float(np.linalg.norm(b))
    if b_norm == 0.0:
        return OracleSolveReport(np.zeros(n), 0, [0.0], True, "bicgstab", true_residual=0.0)
    x = np.zeros(n)
    r = b.copy()
    r_sh = r.copy()
    rho_prev = alpha = omega = 1.0
    v = np.zeros(n)
    p = np.zeros(n)
    history = []
    breakdown = converged = False
    it = 0
    eps = 1e-30
    while it < max_iter:
        rho = float(np.dot(r_sh, r))
        if abs(rho) < eps:
            breakdown = True
            break
        if it == 0:
            p = r.copy()
        else:
            beta = (rho / rho_prev) * (alpha / omega)
            p = r + beta * (p - omega * v)
        v = apply(p)
        denom = float(np.dot(r_sh, v))
        if abs(denom) < eps:
            breakdown = True
            break
        alpha = rho / denom
        s = r - alpha * v
        it += 1
        s_norm = float(np.linalg.norm(s))
        if s_norm / b_norm <= rel_tol:
            x = x + alpha * p
            history.append(s_norm / b_norm)
            converged = True
            break
        t = apply(s)
        tt = float(np.dot(t, t))
        if tt < eps:
            breakdown = True
            break
        omega = float(np.dot(t, s)) / tt
        if abs(omega) < eps:
            breakdown = True
            break
        x = x + alpha * p + omega * s
        r = s - omega * t
        rho_prev = rho
        rel = float(np.linalg.norm(r)) / b_norm
        history.append(rel)
        if rel <= rel_tol:
            converged = True
            break
    true_rel = float(np.linalg.norm(b - apply(x))) / b_norm
    if converged:
        converged = true_rel <= 10.0 * rel_tol
    if not history:
        history.append(true_rel)
    return OracleSolveReport(x, it, history, converged, "bicgstab", breakdown, true_rel)
