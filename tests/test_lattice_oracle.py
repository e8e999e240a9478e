"""CPU tests of the multi-D lattice oracle: reductions to the reference 1D sweep, layout
equivalence, harmonics addition theorem, product setup == oracle setup."""
import math

import numpy as np
import pytest

from paper_2602_21958_b200 import lattice as L
from oracle import lattice as OL
from oracle import rt_oracle as ro


def tiny(nx=6, ny=1, nz=7, n_polar=4, n_az=4, nf=5, **kw):
    return L.lattice_problem(nx, ny, nz, n_polar, n_az, nf, corr_len=2.0, seed=3, **kw)


def test_dipole_addition_theorem():
    omega, w = L.product_quadrature(8, 16)
    Y = L.dipole_harmonics(omega)
    c = np.array(L.DIPOLE_3D_COEFFS)
    lhs = Y.T @ (c[:, None] * Y)
    cosg = omega @ omega.T
    np.testing.assert_allclose(lhs, 1 + 0.5 * (1.5 * cosg ** 2 - 0.5), atol=1e-14)
    Yo, co = OL.real_dipole_harmonics(omega)
    np.testing.assert_allclose(Y, Yo, atol=1e-15)
    assert abs(w.sum() - 4 * math.pi) <= 1e-13
    # normalisation: (1/4pi) sum_a w_a p(W, W_a) = 1
    np.testing.assert_allclose((lhs * w[None, :]).sum(1) / (4 * math.pi), 1.0, atol=1e-13)


def _column_problem(nz=9, nf=4, solver="ie"):
    """Two purely vertical directions: each line is a node column (sx = sy = 0)."""
    p = tiny(nx=3, nz=nz, nf=nf, formal_solver=solver)
    p.omega = np.array([[0.0, 0.0, -1.0], [0.0, 0.0, 1.0]])
    p.dir_w = np.array([2 * math.pi, 2 * math.pi])
    p.ybasis = L.dipole_harmonics(p.omega)
    return p


@pytest.mark.parametrize("solver", ["ie", "exp_linear", "exp_parabolic"])
def test_vertical_lines_reduce_to_reference_1d_sweep(solver):
    p = _column_problem(solver=solver)
    d = OL.desc_from_lattice_problem(p)
    rng = np.random.default_rng(0)
    S = rng.standard_normal((d.n_space, d.n_dirs, d.n_freq))
    out = OL.lattice_transfer(d, S).reshape(p.nz, p.ny, p.nx, 2, p.n_freq)
    chi = p.chi.reshape(p.nz, p.ny, p.nx)
    for i in range(p.nx):
        dt = 0.5 * (chi[1:, 0, i] + chi[:-1, 0, i])          # trapezoid opacity, dz = 1, |mu| = 1
        dtau = p.phi[:, None] * dt[None, :]
        src = S.reshape(p.nz, p.ny, p.nx, 2, p.n_freq)[:, 0, i]
        down = ro.sweep_down(dtau, src[:, 0, :].T, solver=solver).T
        up = ro.sweep_up(dtau, src[:, 1, :].T, solver=solver).T
        np.testing.assert_allclose(out[:, 0, i, 0, :], down, rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(out[:, 0, i, 1, :], up, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("solver", ["ie", "exp_parabolic"])
def test_integer_shift_direction_is_a_selection(solver):
    """sx = 1: lines hit nodes exactly at every layer, T_RC is a 0/1 selection and the
    recursion is the 1D sweep along the node diagonal (periodic wrap in x); for
    exp-parabolic the downwind point of each node is the next node on the diagonal."""
    p = tiny(nx=5, nz=6, nf=3, formal_solver=solver)
    p.omega = np.array([[1 / math.sqrt(2), 0.0, -1 / math.sqrt(2)]])
    p.dir_w = np.array([4 * math.pi])
    p.ybasis = L.dipole_harmonics(p.omega)
    d = OL.desc_from_lattice_problem(p)
    S = np.random.default_rng(1).standard_normal((d.n_space, 1, d.n_freq))
    out = OL.lattice_transfer(d, S).reshape(p.nz, p.nx, p.n_freq)
    chi = p.chi.reshape(p.nz, p.nx)
    Sg = S.reshape(p.nz, p.nx, p.n_freq)
    for lx in range(p.nx):
        cols = [(lx + k) % p.nx for k in range(p.nz)]
        c = np.array([chi[k, cols[k]] for k in range(p.nz)])
        dt = math.sqrt(2) * 0.5 * (c[1:] + c[:-1])
        dtau = p.phi[:, None] * dt[None, :]
        src = np.array([Sg[k, cols[k]] for k in range(p.nz)]).T
        ref = ro.sweep_down(dtau, src, solver=solver).T
        got = np.array([out[k, cols[k]] for k in range(p.nz)])
        np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("ny", [1, 4])
def test_moment_layout_equals_intensity_layout(ny):
    p = tiny(nx=5, ny=ny, nz=6)
    d = OL.desc_from_lattice_problem(p)
    rng = np.random.default_rng(2)
    I = rng.standard_normal(d.n_space * d.n_dirs * d.n_freq)
    u = OL.redistribute(d, OL.moments_of(d, I)).reshape(-1)
    lhs = OL.redistribute(d, OL.moments_of(d, OL.apply_A_intensity(d, I))).reshape(-1)
    np.testing.assert_allclose(OL.apply_A_moments(d, u), lhs, rtol=1e-12, atol=1e-14)
    bI = OL.build_rhs_intensity(d)
    np.testing.assert_allclose(OL.build_rhs_moments(d), OL.redistribute(d, OL.moments_of(d, bI)).reshape(-1),
                               rtol=1e-12, atol=1e-15)


def test_lattice_solution_layouts_agree():
    """Unrestarted GMRES counts agree between layouts and I = Lambda S(u) + b reproduces I."""
    p = tiny(nx=4, ny=1, nz=6, nf=5)
    d = OL.desc_from_lattice_problem(p)
    bI = OL.build_rhs_intensity(d)
    bu = OL.build_rhs_moments(d)
    rI = ro.gmres(lambda v: OL.apply_A_intensity(d, v), bI, rel_tol=1e-11, max_iter=400)
    ru = ro.gmres(lambda v: OL.apply_A_moments(d, v), bu, rel_tol=1e-11, max_iter=400)
    assert rI.converged and ru.converged
    assert abs(rI.iterations - ru.iterations) <= 1
    S = OL.source_from_moments(d, ru.solution)
    I_from_u = OL.lattice_transfer(d, S).reshape(-1) + bI
    assert np.linalg.norm(I_from_u - rI.solution) <= 1e-8 * np.linalg.norm(rI.solution)


def test_stratification_and_field():
    k0 = L.stratified_opacity(65)
    t = np.concatenate([[0], np.cumsum(0.5 * (k0[1:] + k0[:-1]))])
    assert 5e3 < t[-1] < 2e4
    rho = L.lognormal_field((16, 16, 16), 0.5, 4.0, 1)
    g = (np.log(rho) + 0.125) / 0.5
    assert abs(g.std() - 1) < 1e-12 and abs(g.mean()) < 1e-12


# ---------------- short / hybrid characteristics ----------------

def _desc(p, characteristics):
    d = OL.desc_from_lattice_problem(p)
    d.characteristics = characteristics
    return d


@pytest.mark.parametrize("solver", ["ie", "exp_linear", "exp_parabolic"])
def test_short_characteristics_equal_long_on_integer_shift_directions(solver):
    """Vertical and sx = 1 directions: the upwind point of every node is a node, so the
    SC restart is a selection and SC, LC and hybrid coincide."""
    p = tiny(nx=5, nz=8, nf=3, formal_solver=solver)
    s = math.sqrt(0.5)
    p.omega = np.array([[0.0, 0.0, -1.0], [0.0, 0.0, 1.0], [s, 0.0, -s], [-s, 0.0, s]])
    p.dir_w = np.full(4, math.pi)
    p.ybasis = L.dipole_harmonics(p.omega)
    rng = np.random.default_rng(1)
    S = rng.standard_normal((p.n_space, 4, p.n_freq))
    lc = OL.lattice_transfer(_desc(p, "long"), S)
    for mode in ("short", "hybrid"):
        np.testing.assert_allclose(OL.lattice_transfer(_desc(p, mode), S), lc, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("solver", ["ie", "exp_linear", "exp_parabolic"])
def test_short_characteristics_equal_long_for_horizontally_uniform_fields(solver):
    """Horizontally uniform opacity and source: bilinear interpolation is exact, so SC = LC
    for every direction, including grazing ones with several sub-segments per layer."""
    p = tiny(nx=6, ny=4, nz=7, n_polar=8, n_az=6, nf=3, formal_solver=solver)
    chi = p.chi.reshape(p.nz, p.ny, p.nx)
    p.chi = np.repeat(chi[:, :1, :1], p.ny, 1).repeat(p.nx, 2).reshape(-1)
    rng = np.random.default_rng(2)
    S = np.repeat(rng.standard_normal((p.nz, 1, 1, p.n_dirs, p.n_freq)), p.ny, 1).repeat(p.nx, 2)
    S = S.reshape(p.n_space, p.n_dirs, p.n_freq)
    lc = OL.lattice_transfer(_desc(p, "long"), S, with_boundary=True)
    sc = OL.lattice_transfer(_desc(p, "short"), S, with_boundary=True)
    np.testing.assert_allclose(sc, lc, rtol=1e-12, atol=1e-14)


def test_hybrid_takes_short_for_steep_and_long_for_grazing_directions():
    p = tiny(nx=6, ny=5, nz=6, n_polar=8, n_az=6, nf=3)
    rng = np.random.default_rng(3)
    S = rng.standard_normal((p.n_space, p.n_dirs, p.n_freq))
    outs = {m: OL.lattice_transfer(_desc(p, m), S) for m in ("long", "short", "hybrid")}
    d = _desc(p, "hybrid")
    steep = [OL.direction_geometry(d, a)[3] == 1 for a in range(p.n_dirs)]
    assert any(steep) and not all(steep)
    for a in range(p.n_dirs):
        ref = outs["short"] if steep[a] else outs["long"]
        np.testing.assert_array_equal(outs["hybrid"][:, a, :], ref[:, a, :])
    # on a heterogeneous field the two characteristics are different discretisations
    assert np.abs(outs["short"] - outs["long"]).max() > 1e-6


def test_short_characteristics_constant_source_relaxes_to_source():
    """A constant source with matching inflow is a fixed point of the exact transfer; the SC
    restart (rows of the bilinear stencil sum to one) keeps it one to rounding."""
    p = tiny(nx=5, ny=3, nz=6, n_polar=8, n_az=4, nf=3, formal_solver="exp_linear")
    p.inflow_top = np.full(p.n_freq, 0.7)
    p.inflow_bottom = np.full(p.n_freq, 0.7)
    S = np.full((p.n_space, p.n_dirs, p.n_freq), 0.7)
    out = OL.lattice_transfer(_desc(p, "short"), S, with_boundary=True)
    np.testing.assert_allclose(out, 0.7, rtol=1e-13)


def test_characteristics_validation():
    p = tiny()
    with pytest.raises(ValueError):
        OL.lattice_transfer(_desc(p, "medium"), np.zeros((p.n_space, p.n_dirs, p.n_freq)))


def test_exp_parabolic_constant_source_is_a_fixed_point():
    """Kunasz-Auer weights sum to e0, so a constant source with matching inflow stays
    constant through every sub-segment, layer crossing and downwind lookup."""
    for chars in ("long", "short"):
        p = tiny(nx=5, ny=3, nz=6, n_polar=8, n_az=4, nf=3, formal_solver="exp_parabolic")
        p.inflow_top = np.full(p.n_freq, 0.3)
        p.inflow_bottom = np.full(p.n_freq, 0.3)
        S = np.full((p.n_space, p.n_dirs, p.n_freq), 0.3)
        out = OL.lattice_transfer(_desc(p, chars), S, with_boundary=True)
        np.testing.assert_allclose(out, 0.3, rtol=1e-12)


def test_exp_parabolic_differs_from_linear_only_through_curvature():
    """A source linear in depth along vertical lines in a uniform medium: parabolic and
    linear interpolation agree (both exact); on a random source they differ."""
    p = _column_problem(nz=9, nf=3, solver="exp_parabolic")
    p.chi = np.ones_like(p.chi)
    d_par = OL.desc_from_lattice_problem(p)
    d_lin = OL.desc_from_lattice_problem(p)
    d_lin.formal_solver = "exp_linear"
    z = np.arange(p.nz, dtype=float)
    S_lin = np.broadcast_to((2.0 + 0.5 * z)[:, None, None, None, None],
                            (p.nz, p.ny, p.nx, 2, p.n_freq)).reshape(p.n_space, 2, p.n_freq).copy()
    np.testing.assert_allclose(OL.lattice_transfer(d_par, S_lin), OL.lattice_transfer(d_lin, S_lin),
                               rtol=1e-12, atol=1e-14)
    S_rnd = np.random.default_rng(5).standard_normal((p.n_space, 2, p.n_freq))
    assert np.abs(OL.lattice_transfer(d_par, S_rnd) - OL.lattice_transfer(d_lin, S_rnd)).max() > 1e-6


def test_lattice_oracle_matches_reference_multidim_long_characteristics():
    """Pinned against the reference's own 2D long characteristics (R/multidim.py: trace_rays,
    build_interpolators, build_transfer_2d, sweep_lines) on the configuration where both
    discretisations coincide (tests/golden/make_multidim_golden.py): homogeneous transfer of
    three seeded per-ray sources and the boundary term of constant inflows."""
    from tests import _multidim_golden as MG

    z = MG.load()
    d = OL.desc_from_lattice_problem(MG.column_problem(z))
    for S, ref in zip(z["source"], z["lambda"]):
        out = OL.lattice_transfer(d, S.reshape(-1, 2, 1))
        np.testing.assert_allclose(out.reshape(ref.shape), ref, rtol=1e-13, atol=1e-15)
    bnd = OL.lattice_transfer(d, np.zeros((d.n_space, 2, 1)), with_boundary=True)
    np.testing.assert_allclose(bnd.reshape(z["boundary"].shape), z["boundary"], rtol=1e-13, atol=1e-15)
