"""Known-answer and reduction tests that pin the oracle EXTENSIONS (no reference code exists
for the PRD matrix, the exponential formal solvers or the C port) -- CPU only."""
import math

import numpy as np
import pytest

import paper_2602_21958_b200 as P
from paper_2602_21958_b200 import configs
from paper_2602_21958_b200.redistribution import prd_matrix, row_normalisation_error
from oracle import cport
from oracle import rt_oracle as ro
from tests import _golden as G
from tests._problems import oracle_desc, rel_l2


# ---------------- exponential integrator weights ----------------

def _exact_e(d):
    """e0, e1, e2 to 50 digits via the closed forms in decimal arithmetic."""
    from decimal import Decimal, getcontext

    getcontext().prec = 60
    dd = Decimal(d)
    e0 = 1 - (-dd).exp()
    e1 = dd - e0
    e2 = dd * dd - 2 * e1
    return float(e0), float(e1), float(e2)


@pytest.mark.parametrize("d", [1e-12, 1e-6, 1e-3, 0.02, 0.0499, 0.05, 0.2, 0.4999, 0.5, 1.0, 3.0, 30.0])
def test_exp_weights_accuracy(d):
    att, e0, e1, e2 = ro.exp_weights(np.array([d]))
    x0, x1, x2 = _exact_e(d)
    # relative accuracy: ~1 ulp in the series branch, cancellation-limited (eps / (e1/d)) above it
    tol1 = 4e-16 if d < ro.EXP_SERIES_THRESHOLD else 4e-16 * max(1.0, d / x1)
    assert abs(e0[0] - x0) <= 4e-16 * x0
    assert abs(e1[0] - x1) <= tol1 * x1
    assert abs(e2[0] - x2) <= 4 * tol1 * max(1.0, d * d / x2) * x2
    assert abs(att[0] - math.exp(-d)) <= 2e-16 * max(1.0, 1 / math.exp(-d)) * math.exp(-d) + 1e-16


def test_exp_weight_branches_are_continuous():
    for t in (ro.EXP_SERIES_THRESHOLD, 0.5):
        lo = ro.exp_weights(np.array([np.nextafter(t, 0)]))
        hi = ro.exp_weights(np.array([t]))
        for a, b in zip(lo, hi):
            assert abs(a[0] - b[0]) <= 5e-13 * max(abs(b[0]), 1e-300)   # e2 closed form cancels ~1e-13 at 0.05


def _ray_problem(dtau, src, solver, acc0=0.0):
    return ro.sweep_down(np.asarray(dtau)[None, :], np.asarray(src)[None, :], [acc0], solver)[0]


def _exact_solution(tau, coeffs, i0):
    """I(tau) for S(t) = c0 + c1 t + c2 t^2 along the ray, I(0) = i0."""
    c0, c1, c2 = coeffs
    # int_0^tau S(t) e^{-(tau-t)} dt  for polynomial S
    p0 = c0 + c1 * tau + c2 * tau * tau
    p1 = c1 + 2 * c2 * tau
    p2 = 2 * c2
    return p0 - p1 + p2 - (c0 - c1 + p2) * math.exp(-tau) + i0 * math.exp(-tau)


@pytest.mark.parametrize("solver,coeffs", [("exp_linear", (1.3, 0.7, 0.0)), ("exp_parabolic", (0.4, -0.3, 0.25)),
                                           ("exp_linear", (2.0, 0.0, 0.0))])
def test_exponential_solvers_exact_for_polynomial_source(solver, coeffs):
    rng = np.random.default_rng(3)
    dtau = np.concatenate([rng.uniform(1e-4, 0.04, 10), rng.uniform(0.05, 3.0, 20)])
    tau = np.concatenate([[0.0], np.cumsum(dtau)])
    S = coeffs[0] + coeffs[1] * tau + coeffs[2] * tau * tau
    out = _ray_problem(dtau, S, solver, acc0=0.9)
    exact = np.array([_exact_solution(t, coeffs, 0.9) for t in tau])
    # parabolic falls back to linear on the last segment; exact only where the source is linear there
    check = slice(None) if (solver == "exp_linear" or coeffs[2] == 0) else slice(0, -1)
    np.testing.assert_allclose(out[check], exact[check], rtol=2e-13, atol=2e-14)


def test_constant_source_relaxes_to_source():
    dtau = np.full(50, 0.7)
    out = _ray_problem(dtau, np.full(51, 3.0), "exp_linear", acc0=0.0)
    tau = np.arange(51) * 0.7
    np.testing.assert_allclose(out, 3.0 * (1 - np.exp(-tau)), rtol=1e-14, atol=1e-15)


def test_ie_boundary_term_has_no_overflow():
    """build_transfer's cumprod overflows at tau ~ 1e6 (R/transfer.py:97-99); the recursion must not."""
    d = oracle_desc(configs.slab_problem(2, n_angles=8, n_freq=33))
    d.inflow = np.ones_like(d.inflow)
    b = ro.boundary_term(d)
    assert np.all(np.isfinite(b)) and b.max() <= 1.0 and b.min() >= 0.0


# ---------------- PRD matrix ----------------

@pytest.mark.parametrize("nf,xmax,a", [(31, 5.0, 0.5), (41, 5.0, 1.0), (512, 8.0, 0.5)])
def test_prd_matrix_conserves_photons_and_is_symmetric(nf, xmax, a):
    x, w = ro.trapezoid(nf, -xmax, xmax)
    phi = ro.gaussian_profile(x)
    R = ro.prd_matrix(x, w, phi, a)
    assert np.max(np.abs(R @ w / phi - 1)) <= 2e-15
    assert np.max(np.abs(R - R.T)) <= 1e-16 * np.abs(R).max() * 10
    assert np.all(R >= 0)
    # product-side builder gives the same matrix
    R2 = prd_matrix(x, w, phi, a)
    assert np.max(np.abs(R2 - R)) <= 1e-15 * np.abs(R).max()
    assert row_normalisation_error(R2, w, phi) <= 2e-15


def test_prd_marginal_of_unnormalised_ri_is_profile():
    """Continuous identity behind the choice of R_I: int 1/2 erfc(max(|x|,|x'|)) dx' = phi(x)."""
    xs = np.linspace(-6, 6, 24001)
    h = xs[1] - xs[0]
    for x0 in (0.0, 0.7, 1.9):
        vals = 0.5 * np.vectorize(math.erfc)(np.maximum(abs(x0), np.abs(xs)))
        integral = h * (vals.sum() - 0.5 * (vals[0] + vals[-1]))
        assert abs(integral - math.exp(-x0 * x0) / math.sqrt(math.pi)) <= 1e-6


# ---------------- reductions of the dipole x PRD kernel to reference kernels ----------------

def test_dipole_prd_with_flat_r_equals_reference_legendre_kernel():
    z = G.load()
    key = "cfg1_legendre"
    d = G.desc(key)
    Y, c, _ = ro.legendre_as_general((1.0, 0.0, 0.5), d.mu, d.n_freq)
    d.ybasis, d.coeffs, d.R = Y, c, np.ones((d.n_freq, d.n_freq))
    for v, ref in zip(z[f"{key}/v"], z[f"{key}/Av"]):
        assert rel_l2(ro.apply_A(d, v), ref) <= 1e-13


def test_dipole_prd_with_crd_r_equals_reference_crd_kernel():
    z = G.load()
    key = "cfg1_crd"
    d = G.desc(key)
    d.ybasis, d.coeffs, d.R = np.ones((1, d.n_angles)), np.ones(1), np.outer(d.phi, d.phi)
    for v, ref in zip(z[f"{key}/v"], z[f"{key}/Av"]):
        assert rel_l2(ro.apply_A(d, v), ref) <= 1e-13


def test_dense_operator_matches_matrix_free_on_tiny_prd_problem():
    p = configs.slab_problem(1, n_space=6, n_angles=4, n_freq=5)
    d = oracle_desc(p)
    dense = ro.materialize(lambda v: ro.apply_A(d, v), d.n_total)
    psi = ro.psi_dipole_prd(d.ybasis, d.coeffs, d.R)
    w = np.repeat(d.ang_w, d.n_freq) * np.tile(d.freq_w, d.n_angles)
    lam = ro.materialize(lambda v: ro.apply_transfer(d, v), d.n_total)
    sig = np.zeros_like(lam)
    nr = d.n_rays
    for i in range(d.n_space):
        sig[i * nr:(i + 1) * nr, i * nr:(i + 1) * nr] = d.gamma[i][:, None] * psi * w[None, :]
    np.testing.assert_allclose(dense, np.eye(d.n_total) - lam @ sig, atol=1e-14)


# ---------------- product host setup == oracle setup ----------------

def test_product_setup_matches_oracle_setup():
    p = configs.slab_problem(1)
    g = p.grid
    x, w = ro.gauss_legendre(8, -1.0, 0.0)
    np.testing.assert_array_equal(g.mu_nodes[:8], x)
    np.testing.assert_array_equal(g.angular_weights[:8], w)
    nu, fw = ro.trapezoid(31, -5.0, 5.0)
    np.testing.assert_array_equal(g.nu_nodes, nu)
    np.testing.assert_array_equal(g.frequency_weights, fw)
    Y, c, R = P.separable_form(p.scattering.kernel, g)
    assert Y.shape == (2, 16) and list(c) == [1.0, 0.5]     # l = 1 dropped (coefficient 0)
    np.testing.assert_array_equal(Y[1], ro.legendre_basis(2, g.mu_nodes)[2])


# ---------------- C port == numpy oracle ----------------

@pytest.mark.parametrize("fs", ["ie", "exp_linear", "exp_parabolic"])
def test_c_port_matches_numpy_oracle(fs):
    p = configs.slab_problem(1, formal_solver=fs, n_space=60, n_freq=21)
    d = oracle_desc(p)
    v = np.random.default_rng(1).standard_normal(d.n_total)
    assert rel_l2(cport.SlabPort(d).apply_A(v), ro.apply_A(d, v)) <= 1e-14


# ---------------- GMRES oracle vs LU ----------------

def test_oracle_gmres_matches_lu_on_prd_problem():
    p = configs.slab_problem(1, n_space=12, n_angles=4, n_freq=7)
    d = oracle_desc(p)
    A = ro.materialize(lambda v: ro.apply_A(d, v), d.n_total)
    b = ro.build_rhs(d)
    rep = ro.gmres(lambda v: ro.apply_A(d, v), b, rel_tol=1e-12, max_iter=d.n_total)
    assert rep.converged
    np.testing.assert_allclose(rep.solution, np.linalg.solve(A, b), rtol=1e-9, atol=1e-12)
