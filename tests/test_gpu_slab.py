"""GPU parity of the 1D (I - Lambda Sigma) path against the reference goldens and the oracle.

Tolerance (BASELINE north_star): matvec <= 1e-11 relative L2 against the CPU
oracle on identical seeded inputs; GMRES iterations within +-1 (unrestarted)
and solution within 1e-7 relative.
"""
import numpy as np
import pytest

import paper_2602_21958_b200 as P
from paper_2602_21958_b200 import configs
from oracle import rt_oracle as ro
from tests import _golden as G
from tests._problems import oracle_desc, product_from_golden, rel_l2

pytestmark = pytest.mark.gpu

MATVEC_TOL = 1e-11


@pytest.mark.parametrize("key", G.CASES)
def test_operator_pieces_match_reference_goldens(key):
    z = G.load()
    p = product_from_golden(key)
    for v, sv, lv, av in zip(z[f"{key}/v"], z[f"{key}/Sigma_v"], z[f"{key}/Lambda_v"], z[f"{key}/Av"]):
        assert rel_l2(P.apply_A(p, v), av) <= MATVEC_TOL
        assert rel_l2(P.apply_scattering(p.scattering, v), sv) <= MATVEC_TOL
        assert rel_l2(P.apply_transfer(p.transfer, v), lv) <= MATVEC_TOL


@pytest.mark.parametrize("key", G.CASES)
def test_rhs_matches_reference_goldens(key):
    z = G.load()
    p = product_from_golden(key)
    np.testing.assert_allclose(P.build_rhs(p), z[f"{key}/rhs"], rtol=1e-12, atol=1e-15)


GOLDEN_GMRES_KEYS = ["mono", "coherent", "crd", "log_legendre", "log_crd", "cfg1_legendre", "cfg1_crd"]


def iteration_band(key, case):
    """Accepted iteration counts: the golden +-1 (north star) for unrestarted GMRES; for
    restarted GMRES the reference's OWN spread under one-ulp perturbations of b (measured by
    running the unmodified reference, tests/golden/make_gmres_bands.py), widened by +-1.
    E.g. cfg1_crd GMRES(30): golden 738, reference band 709..741."""
    lo = hi = case["iterations"]
    if case["restart"] is not None:
        its = G.gmres_band(key, case["name"])
        lo, hi = min(lo, int(its.min())), max(hi, int(its.max()))
    return lo - 1, hi + 1


@pytest.mark.parametrize("key", GOLDEN_GMRES_KEYS)
@pytest.mark.parametrize("orth", [None, "cgs2"], ids=["reference_mgs", "cgs2"])
def test_gmres_matches_reference_goldens(key, orth):
    """The reference's own Arnoldi (MGS, or MGS2 with reorthogonalize, the golden's setting) and
    the fused CGS2: iteration count within the band above, history prefix and solution."""
    p = product_from_golden(key)
    for case in G.gmres_cases(key):
        cfg = P.SolveConfig(rel_tol=case["rel_tol"], max_iter=case["max_iter"], restart=case["restart"],
                            reorthogonalize=case["reorthogonalize"], orthogonalization=orth)
        rep = P.gmres(p, case["b"], cfg)
        assert rep.converged == case["converged"]
        lo, hi = iteration_band(key, case)
        assert lo <= rep.iterations <= hi, (case["name"], rep.iterations, case["iterations"], lo, hi)
        k = min(len(rep.residual_history), len(case["history"]), 100)
        np.testing.assert_allclose(rep.residual_history[:k], case["history"][:k], rtol=1e-8, atol=1e-13)
        assert rel_l2(rep.solution, case["solution"]) <= 1e-7


@pytest.mark.parametrize("fs", ["ie", "exp_linear", "exp_parabolic"])
def test_cfg1_dipole_prd_matvec_matches_oracle(fs):
    p = configs.slab_problem(1, formal_solver=fs)
    d = oracle_desc(p)
    rng = np.random.default_rng(21958 + 1)
    for _ in range(3):
        v = rng.standard_normal(p.n_total)
        assert rel_l2(P.apply_A(p, v), ro.apply_A(d, v)) <= MATVEC_TOL
    assert rel_l2(P.build_rhs(p), ro.build_rhs(d)) <= MATVEC_TOL


@pytest.mark.parametrize("fs", ["ie", "exp_linear", "exp_parabolic"])
def test_cfg2_full_size_matvec_matches_oracle(fs):
    p = configs.slab_problem(2, formal_solver=fs)
    d = oracle_desc(p)
    v = np.random.default_rng(21958 + 2).standard_normal(p.n_total)
    assert rel_l2(P.apply_A(p, v), ro.apply_A(d, v)) <= MATVEC_TOL


def test_torch_tensor_path_equals_numpy_path():
    import torch

    p = configs.slab_problem(1)
    v = np.random.default_rng(3).standard_normal(p.n_total)
    yt = P.apply_A(p, torch.from_numpy(v).cuda())
    assert yt.is_cuda
    np.testing.assert_array_equal(yt.cpu().numpy(), P.apply_A(p, v))


def test_gamma_zero_gives_identity():
    p = configs.slab_problem(1)
    p.scattering.gamma_table = np.zeros_like(p.scattering.gamma_table)
    p.invalidate()
    v = np.random.default_rng(4).standard_normal(p.n_total)
    np.testing.assert_array_equal(P.apply_A(p, v), v)


def test_linearity_cfg2():
    import torch

    p = configs.slab_problem(2)
    rng = np.random.default_rng(5)
    u = torch.from_numpy(rng.standard_normal(p.n_total)).cuda()
    w = torch.from_numpy(rng.standard_normal(p.n_total)).cuda()
    lhs = P.apply_A(p, 2.5 * u - 1.5 * w)
    rhs = 2.5 * P.apply_A(p, u) - 1.5 * P.apply_A(p, w)
    assert float(torch.linalg.vector_norm(lhs - rhs) / torch.linalg.vector_norm(rhs)) <= 1e-13


def test_length_mismatch_raises_value_error():
    p = configs.slab_problem(1)
    with pytest.raises(ValueError):
        P.apply_A(p, np.zeros(11))


def test_cfg1_gmres_unrestarted_matches_oracle():
    p = configs.slab_problem(1)
    d = oracle_desc(p)
    b = ro.build_rhs(d)
    ref = ro.gmres(lambda v: ro.apply_A(d, v), b, rel_tol=1e-8, max_iter=2000)
    rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=2000))
    assert rep.converged and ref.converged
    assert abs(rep.iterations - ref.iterations) <= 1
    np.testing.assert_allclose(rep.residual_history[:100], ref.residual_history[:100], rtol=1e-9, atol=1e-14)
    assert rel_l2(rep.solution, ref.solution) <= 1e-7


def test_callable_apply_path_matches_native_path():
    p = configs.slab_problem(1)
    b = P.build_rhs(p)
    cfg = P.SolveConfig(rel_tol=1e-8, max_iter=300)
    native = P.gmres(p, b, cfg)
    cb = P.gmres(lambda v: P.apply_A(p, v), b, cfg)
    assert native.iterations == cb.iterations
    np.testing.assert_array_equal(native.solution, cb.solution)


def test_bicgstab_matches_oracle_on_golden_crd():
    p = product_from_golden("crd")
    d = oracle_desc(p)
    b = ro.build_rhs(d)
    ref = ro.bicgstab(lambda v: ro.apply_A(d, v), b, rel_tol=1e-12, max_iter=500)
    rep = P.bicgstab(P.operator(p), b, P.SolveConfig(method="bicgstab", rel_tol=1e-12, max_iter=500))
    assert rep.converged == ref.converged
    assert abs(rep.iterations - ref.iterations) <= 1
    assert rel_l2(rep.solution, ref.solution) <= 1e-7


@pytest.mark.parametrize("fs", ["ie", "exp_linear"])
def test_cp_async_fallback_sweep_matches_tma_sweep(fs):
    """The generic (non-TMA) sweep kernel and the TMA kernel agree to rounding, and both
    match the oracle."""
    p = configs.slab_problem(1, formal_solver=fs)
    v = np.random.default_rng(9).standard_normal(p.n_total)
    y_tma = P.apply_A(p, v)
    p.device().set_tuning("disable_tma", 1)
    y_gen = P.apply_A(p, v)
    assert rel_l2(y_gen, y_tma) <= 1e-14
    assert rel_l2(y_gen, ro.apply_A(oracle_desc(p), v)) <= MATVEC_TOL


def test_unaligned_vector_takes_the_cp_async_sweep():
    """A device x that is not 16-byte aligned (TMA needs 16) is swept by the cp.async kernel
    (decided per call, never a silent fallback after a failed launch)."""
    import torch

    p = configs.slab_problem(1, n_space=40, n_angles=8, n_freq=11)
    v = np.random.default_rng(2).standard_normal(p.n_total)
    buf = torch.empty(p.n_total + 1, dtype=torch.float64, device="cuda")
    buf[1:] = torch.from_numpy(v).cuda()
    y = P.apply_A(p, buf[1:])
    assert rel_l2(y.cpu().numpy(), ro.apply_A(oracle_desc(p), v)) <= MATVEC_TOL


@pytest.mark.parametrize("fs", ["exp_linear", "exp_parabolic"])
@pytest.mark.parametrize("shape", [(2000, 64, 512), (37, 8, 256), (6, 4, 128)])
def test_exponential_sweeps_match_oracle(fs, shape):
    """The exponential TMA sweeps (branch-free range-reduced weights) against the oracle's
    three-branch weights, up to the cfg2 full size."""
    ns, na, nf = shape
    p = configs.slab_problem(2, formal_solver=fs, n_space=ns, n_angles=na, n_freq=nf)
    v = np.random.default_rng(ns + 1).standard_normal(p.n_total)
    assert rel_l2(P.apply_A(p, v), ro.apply_A(oracle_desc(p), v)) <= MATVEC_TOL


@pytest.mark.parametrize("shape", [(37, 6, 5), (64, 12, 130), (50, 4, 257), (9, 2, 1)])
def test_odd_shapes_match_oracle(shape):
    """Ragged shapes: odd N_nu (TMA pitch padding), N_nu > 128 with a partial tile, mono (N_nu = 1)."""
    ns, na, nf = shape
    for fs in ("ie", "exp_linear", "exp_parabolic"):
        p = configs.slab_problem(1, formal_solver=fs, n_space=ns, n_angles=na, n_freq=max(nf, 2))
        d = oracle_desc(p)
        v = np.random.default_rng(ns).standard_normal(p.n_total)
        assert rel_l2(P.apply_A(p, v), ro.apply_A(d, v)) <= MATVEC_TOL


@pytest.mark.parametrize("shape", [(101, 20, 256), (29, 16, 128), (3, 8, 384), (57, 64, 512), (2000, 6, 512)])
def test_fused_sigma_shapes_match_oracle(shape):
    """Shapes the fused moments+redistribution kernel takes (n_freq = 128 CN, two moments):
    partial M blocks, an angle count off the 16-unroll, a single space point, CN = 1..4."""
    ns, na, nf = shape
    p = configs.slab_problem(2, n_space=ns, n_angles=na, n_freq=nf)
    d = oracle_desc(p)
    v = np.random.default_rng(ns + nf).standard_normal(p.n_total)
    assert rel_l2(P.apply_A(p, v), ro.apply_A(d, v)) <= MATVEC_TOL


def test_fused_sigma_equals_unfused_pair():
    """cfg2 full size: the fused kernel and the K2a + K2b pair (and the 8-byte moment kernel)
    agree to rounding."""
    p = configs.slab_problem(2)
    v = np.random.default_rng(5).standard_normal(p.n_total)
    y_fused = P.apply_A(p, v)
    p.device().set_tuning("sigma_unfused", 1)
    y_pair = P.apply_A(p, v)
    assert rel_l2(y_fused, y_pair) <= 1e-14
    p.device().set_tuning("moments_scalar", 1)
    assert rel_l2(P.apply_A(p, v), y_pair) <= 1e-14


@pytest.mark.parametrize("ns", [2, 3, 5, 9])
@pytest.mark.parametrize("fs", ["ie", "exp_linear", "exp_parabolic"])
def test_few_depth_points_match_oracle(ns, fs):
    """Slabs shorter than one pipeline stage (and a first/last stage edge in one): the TMA
    sweeps' boundary handling and the exp-parabolic closing step."""
    p = configs.slab_problem(1, formal_solver=fs, n_space=ns, n_angles=8, n_freq=128)
    d = oracle_desc(p)
    v = np.random.default_rng(ns).standard_normal(p.n_total)
    assert rel_l2(P.apply_A(p, v), ro.apply_A(d, v)) <= MATVEC_TOL


def test_reduced_cfg2_gmres_history_prefix_matches_oracle():
    """cfg2 construction at N_z = 300, 16 mu, 64 nu: first 60 history entries within 1e-9
    (the sharp GMRES parity check), solution within 1e-7."""
    p = configs.slab_problem(2, n_space=300, n_angles=16, n_freq=64)
    d = oracle_desc(p)
    b = ro.build_rhs(d)
    cfg = dict(rel_tol=1e-8, max_iter=60, restart=30)
    ref = ro.gmres(lambda v: ro.apply_A(d, v), b, **cfg)
    rep = P.gmres(p, b, P.SolveConfig(**cfg))
    k = min(len(ref.residual_history), len(rep.residual_history))
    np.testing.assert_allclose(rep.residual_history[:k], ref.residual_history[:k], rtol=1e-9, atol=1e-15)
    assert rep.iterations == ref.iterations
    assert rel_l2(rep.solution, ref.solution) <= 1e-7


def test_source_function_and_boundary_match_oracle():
    p = configs.slab_problem(1)
    p.transfer.inflow = np.random.default_rng(2).uniform(0, 1, p.grid.n_rays)
    d = oracle_desc(p)
    I = np.random.default_rng(8).standard_normal(p.n_total)
    assert rel_l2(P.source_function(p, I), ro.source_function(d, I)) <= MATVEC_TOL
    assert rel_l2(P.boundary_term(p.transfer).values, ro.boundary_term(d)) <= MATVEC_TOL
    assert rel_l2(P.build_rhs(p), ro.build_rhs(d)) <= MATVEC_TOL


def test_spectral_radius_estimate_matches_oracle_power_iteration():
    p = configs.slab_problem(1, n_space=40, n_angles=8, n_freq=11)
    d = oracle_desc(p)
    rng = np.random.default_rng(12345)
    v = rng.standard_normal(d.n_total)
    v /= np.linalg.norm(v)
    ratios = []
    for _ in range(30):
        w = v - ro.apply_A(d, v)
        nrm = np.linalg.norm(w)
        ratios.append(nrm)
        v = w / nrm
    ref = float(np.exp(np.mean(np.log(ratios[-5:]))))
    assert abs(P.spectral_radius_estimate(p, iters=30) - ref) <= 1e-9 * ref


def test_materialize_A_matches_oracle_dense():
    p = configs.slab_problem(1, n_space=6, n_angles=4, n_freq=5)
    d = oracle_desc(p)
    np.testing.assert_allclose(P.materialize_A(p), ro.materialize(lambda v: ro.apply_A(d, v), d.n_total),
                               atol=1e-13)


def test_field_vector_ray_major_round_trip():
    p = configs.slab_problem(1, n_space=10, n_angles=4, n_freq=3)
    v = np.random.default_rng(1).standard_normal(p.n_total)
    fv = P.permute(p.grid, P.FieldVector(v, P.Ordering.SPACE_MAJOR), P.Ordering.RAY_MAJOR)
    out = P.apply_transfer(p.transfer, fv)
    assert out.ordering is P.Ordering.RAY_MAJOR
    back = P.permute(p.grid, out, P.Ordering.SPACE_MAJOR).values
    np.testing.assert_allclose(back, P.apply_transfer(p.transfer, v), rtol=1e-15, atol=1e-16)


def test_cfg2_full_size_gmres_history_prefix_matches_oracle():
    """Full cfg2 (N = 65.5M): the first 12 GMRES(30) iterations agree with the oracle GMRES
    (reference MGS control flow) driving the C/OpenMP port's matvec (itself pinned to the numpy
    oracle in tests/test_oracle_extensions.py)."""
    from oracle import cport

    p = configs.slab_problem(2)
    d = oracle_desc(p)
    port = cport.SlabPort(d)
    b = np.random.default_rng(21958).standard_normal(p.n_total)
    ref = ro.gmres(port.apply_A, b, rel_tol=1e-30, max_iter=12, restart=30)
    rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-30, max_iter=12, restart=30))
    np.testing.assert_allclose(rep.residual_history, ref.residual_history, rtol=1e-9)
    assert rel_l2(rep.solution, ref.solution) <= 1e-7


def test_apply_A_batch_matches_single_calls():
    import torch

    p = configs.slab_problem(2, n_space=200, n_angles=16, n_freq=130)
    rng = np.random.default_rng(4)
    xs = [torch.from_numpy(rng.standard_normal(p.n_total)).pin_memory().numpy() for _ in range(5)]
    ys = P.apply_A_batch(p, xs)
    for x, y in zip(xs, ys):
        np.testing.assert_array_equal(y, P.apply_A(p, x))


@pytest.mark.parametrize("fs", ["ie", "exp_linear"])
@pytest.mark.parametrize("shape", [(1, None), (2, dict(n_space=300, n_angles=16, n_freq=130)), (2, None)])
def test_moment_layout_matvec_matches_oracle(fs, shape):
    cfg, kw = shape
    p = configs.slab_problem(cfg, formal_solver=fs, layout="moments", **(kw or {}))
    d = oracle_desc(p)
    u = np.random.default_rng(31).standard_normal(p.n_total)
    assert rel_l2(P.apply_A(p, u), ro.apply_A_moments(d, u)) <= MATVEC_TOL
    if cfg == 1:
        assert rel_l2(P.build_rhs(p), ro.build_rhs_moments(d)) <= MATVEC_TOL


def test_moment_layout_solve_reproduces_intensity_solve():
    """Unrestarted GMRES: same iteration count (+-1) in both layouts, and I(u*) equals the
    intensity-layout solution."""
    pi = configs.slab_problem(1)
    pm = configs.slab_problem(1, layout="moments")
    cfg = P.SolveConfig(rel_tol=1e-10, max_iter=500)
    ri = P.gmres(pi, P.build_rhs(pi), cfg)
    rm = P.gmres(pm, P.build_rhs(pm), cfg)
    assert ri.converged and rm.converged
    assert abs(ri.iterations - rm.iterations) <= 1
    I = P.intensity_from_moments(pm, rm.solution)
    assert rel_l2(I, ri.solution) <= 1e-8
    d = oracle_desc(pm)
    assert rel_l2(I, ro.intensity_from_moments(d, rm.solution)) <= 1e-11


def test_matvec_and_gmres_are_bitwise_reproducible():
    """Fixed-order reductions everywhere (fused sigma cluster hand-off, CGS2 block sums, no
    atomics): repeated runs give identical bits (run-to-run reproducibility)."""
    import torch

    p = configs.slab_problem(2)
    x = torch.from_numpy(np.random.default_rng(11).standard_normal(p.n_total)).cuda()
    y1 = P.apply_A(p, x).cpu().numpy()
    y2 = P.apply_A(p, x).cpu().numpy()
    np.testing.assert_array_equal(y1, y2)
    q = configs.slab_problem(1)
    b = P.build_rhs(q)
    r1 = P.gmres(q, b, P.SolveConfig(rel_tol=1e-8, max_iter=200, restart=30))
    r2 = P.gmres(q, b, P.SolveConfig(rel_tol=1e-8, max_iter=200, restart=30))
    assert r1.iterations == r2.iterations
    np.testing.assert_array_equal(r1.residual_history, r2.residual_history)
    np.testing.assert_array_equal(r1.solution, r2.solution)


def test_random_configurations_match_dense_oracle_and_lu():
    """Acceptance-criterion-6 pattern (T/test_acceptance.py:188-242) on the device path: 20
    seeded random small problems (reference presets and the dipole x PRD kernel, all three formal
    solvers); the dense matrix comes from the CPU oracle, the device matvec must agree to 1e-12
    and the native GMRES solution with the LU solve to 1e-8."""
    from paper_2602_21958_b200 import presets

    rng = np.random.default_rng(20260810)
    for trial in range(20):
        kind = rng.choice(["mono", "coherent", "crd", "prd"])
        if kind == "mono":
            p = presets.build("mono", n_space=int(rng.integers(5, 40)), n_angles=int(rng.choice([4, 8, 12])))
        elif kind in ("coherent", "crd"):
            p = presets.build(kind, n_space=int(rng.integers(4, 15)), n_angles=int(rng.choice([4, 8])),
                              n_freq=int(rng.integers(3, 12)))
        else:
            p = configs.slab_problem(1, formal_solver=str(rng.choice(["ie", "exp_linear", "exp_parabolic"])),
                                     n_space=int(rng.integers(4, 20)), n_angles=int(rng.choice([4, 8])),
                                     n_freq=int(rng.integers(3, 12)))
        n = p.n_total
        if n > 1500:
            continue
        d = oracle_desc(p)
        dense = np.stack([ro.apply_A(d, e) for e in np.eye(n)], axis=1)
        for _ in range(3):
            v = rng.standard_normal(n)
            assert rel_l2(P.apply_A(p, v), dense @ v) <= 1e-12, (trial, kind)
        b = rng.standard_normal(n)
        rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-13, max_iter=n))
        x = np.linalg.solve(dense, b)
        assert rel_l2(rep.solution, x) <= 1e-8, (trial, kind, rep.iterations)
