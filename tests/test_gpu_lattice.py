"""GPU parity of the multi-D lattice operator (configs 3-5 construction) against the oracle."""
import numpy as np
import pytest

import paper_2602_21958_b200 as P
from paper_2602_21958_b200 import configs
from paper_2602_21958_b200 import lattice as L
from oracle import lattice as OL
from oracle import rt_oracle as ro
from tests._problems import rel_l2

pytestmark = pytest.mark.gpu
MATVEC_TOL = 1e-11

CASES = [  # (nx, ny, nz, n_polar, n_az, n_freq)
    (16, 1, 12, 8, 16, 5),     # 2D slab, cfg3 angular set
    (8, 8, 6, 8, 12, 4),       # 3D box, cfg5 angular set
    (7, 5, 5, 4, 6, 3),        # ragged 3D
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("layout", ["intensity", "moments"])
@pytest.mark.parametrize("fs", ["ie", "exp_linear", "exp_parabolic"])
def test_lattice_matvec_matches_oracle(case, layout, fs):
    nx, ny, nz, npol, naz, nf = case
    p = L.lattice_problem(nx, ny, nz, npol, naz, nf, corr_len=2.0, seed=11, layout=layout, formal_solver=fs)
    d = OL.desc_from_lattice_problem(p)
    rng = np.random.default_rng(nx * 100 + nz)
    for _ in range(2):
        v = rng.standard_normal(p.n_total)
        assert rel_l2(P.apply_A(p, v), OL.apply_A(d, layout, v)) <= MATVEC_TOL
    assert rel_l2(P.build_rhs(p), OL.build_rhs(d, layout)) <= MATVEC_TOL


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("layout", ["intensity", "moments"])
@pytest.mark.parametrize("chars", ["short", "hybrid"])
@pytest.mark.parametrize("fs", ["ie", "exp_linear", "exp_parabolic"])
def test_short_and_hybrid_characteristics_match_oracle(case, layout, chars, fs):
    """Short characteristics (restart at each node's upwind point every layer step) and the
    hybrid (short for steep, long for grazing directions) against the oracle."""
    nx, ny, nz, npol, naz, nf = case
    p = L.lattice_problem(nx, ny, nz, npol, naz, nf, corr_len=2.0, seed=13, layout=layout, formal_solver=fs,
                          characteristics=chars)
    d = OL.desc_from_lattice_problem(p)
    assert d.characteristics == chars
    v = np.random.default_rng(nx + nz).standard_normal(p.n_total)
    assert rel_l2(P.apply_A(p, v), OL.apply_A(d, layout, v)) <= MATVEC_TOL
    assert rel_l2(P.build_rhs(p), OL.build_rhs(d, layout)) <= MATVEC_TOL


def test_hybrid_characteristics_gmres_matches_oracle():
    p = L.lattice_problem(8, 6, 8, 8, 8, 4, corr_len=2.0, seed=7, layout="moments", characteristics="hybrid")
    d = OL.desc_from_lattice_problem(p)
    b = OL.build_rhs(d, "moments")
    ref = ro.gmres(lambda v: OL.apply_A(d, "moments", v), b, rel_tol=1e-8, max_iter=500)
    rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=500))
    assert rep.converged and ref.converged
    assert abs(rep.iterations - ref.iterations) <= 1
    assert rel_l2(rep.solution, ref.solution) <= 1e-7


@pytest.mark.parametrize("layout", ["intensity", "moments"])
def test_lattice_gmres_matches_oracle(layout):
    p = L.lattice_problem(8, 1, 10, 8, 8, 5, corr_len=2.0, seed=5, layout=layout)
    d = OL.desc_from_lattice_problem(p)
    b = OL.build_rhs(d, layout)
    ref = ro.gmres(lambda v: OL.apply_A(d, layout, v), b, rel_tol=1e-8, max_iter=500)
    rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=500))
    assert rep.converged and ref.converged
    assert abs(rep.iterations - ref.iterations) <= 1
    assert rel_l2(rep.solution, ref.solution) <= 1e-7


def test_cfg3_full_size_linearity_and_layout_identity():
    """Size-independent properties at the cfg3 size (256 x 256, 128 dirs, 41 nu)."""
    import torch

    p = L.lattice_problem(256, 1, 256, 8, 16, 41, corr_len=16.0, seed=21958 + 3)
    rng = torch.Generator(device="cuda").manual_seed(3)
    u = torch.randn(p.n_total, dtype=torch.float64, device="cuda", generator=rng)
    w = torch.randn(p.n_total, dtype=torch.float64, device="cuda", generator=rng)
    lhs = P.apply_A(p, 2.0 * u - 0.5 * w)
    rhs = 2.0 * P.apply_A(p, u) - 0.5 * P.apply_A(p, w)
    assert float(torch.linalg.vector_norm(lhs - rhs) / torch.linalg.vector_norm(rhs)) <= 1e-13


def test_lattice_bicgstab_matches_oracle():
    p = L.lattice_problem(6, 1, 8, 4, 8, 5, corr_len=2.0, seed=9, layout="moments")
    d = OL.desc_from_lattice_problem(p)
    b = OL.build_rhs(d, "moments")
    ref = ro.bicgstab(lambda v: OL.apply_A(d, "moments", v), b, rel_tol=1e-9, max_iter=300)
    rep = P.bicgstab(p, b, P.SolveConfig(method="bicgstab", rel_tol=1e-9, max_iter=300))
    assert rep.converged == ref.converged
    assert abs(rep.iterations - ref.iterations) <= 1
    assert rel_l2(rep.solution, ref.solution) <= 1e-7


def test_lattice_rejects_bad_arguments():
    p = L.lattice_problem(4, 1, 4, 4, 4, 3, corr_len=1.0)
    with pytest.raises(ValueError):
        P.apply_A(p, np.zeros(7))
    q = L.lattice_problem(4, 1, 4, 4, 4, 3, corr_len=1.0, formal_solver="exp_cubic")
    with pytest.raises(ValueError):
        q.device()
    r = L.lattice_problem(4, 1, 4, 4, 4, 3, corr_len=1.0, characteristics="medium")
    with pytest.raises(ValueError):
        r.device()


@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_lattice_matvec_matches_oracle(cfg):
    """BASELINE cfg3 (256 x 256 slab, 128 dirs, 41 nu, intensity layout) and cfg4 (64^3, 128 dirs,
    31 nu, moment layout) at full size: one matvec against the numpy oracle (1 - 3 min on the CPU)."""
    p = configs.lattice_config_problem(cfg)
    d = OL.desc_from_lattice_problem(p)
    v = np.random.default_rng(cfg).standard_normal(p.n_total)
    assert rel_l2(P.apply_A(p, v), OL.apply_A(d, p.layout, v)) <= MATVEC_TOL


def test_exp_parabolic_lattice_gmres_matches_oracle():
    p = L.lattice_problem(6, 5, 8, 8, 8, 4, corr_len=2.0, seed=9, layout="moments", formal_solver="exp_parabolic",
                          characteristics="hybrid")
    d = OL.desc_from_lattice_problem(p)
    b = OL.build_rhs(d, "moments")
    ref = ro.gmres(lambda v: OL.apply_A(d, "moments", v), b, rel_tol=1e-8, max_iter=500)
    rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=500))
    assert rep.converged and ref.converged
    assert abs(rep.iterations - ref.iterations) <= 1
    assert rel_l2(rep.solution, ref.solution) <= 1e-7


def test_lattice_matvec_is_bitwise_reproducible():
    """The direction-grouped moment kernel sums its partial moments in a fixed order."""
    import torch

    p = L.lattice_problem(16, 16, 8, 8, 12, 6, corr_len=2.0, seed=2, layout="moments", characteristics="hybrid")
    u = torch.from_numpy(np.random.default_rng(1).standard_normal(p.n_total)).cuda()
    np.testing.assert_array_equal(P.apply_A(p, u).cpu().numpy(), P.apply_A(p, u).cpu().numpy())


@pytest.mark.parametrize("fs", ["ie", "exp_linear", "exp_parabolic"])
@pytest.mark.parametrize("chars", ["long", "hybrid"])
def test_thick_limit_lambda_reproduces_the_source(fs, chars):
    """T/test_multidim.py:115-123 pattern: in an optically thick medium (Delta tau >> 1 per
    cell) the formal solution of a constant source is the source away from the inflow
    boundaries; the device transfer (thermal source path of build_rhs, zero inflow) shows it."""
    p = L.lattice_problem(8, 6, 10, 8, 8, 3, corr_len=2.0, seed=3, layout="intensity", formal_solver=fs,
                          characteristics=chars, t_range=(1e3, 1e6))
    p.inflow_bottom = np.zeros(p.n_freq)
    p.thermal = np.ones_like(p.thermal)
    I = P.build_rhs(p).reshape(p.nz, p.ny, p.nx, p.n_dirs, p.n_freq)
    # line centre (the wings, phi ~ 1e-11, stay optically thin)
    np.testing.assert_allclose(I[2:-2, ..., 1], 1.0, rtol=1e-4)
    np.testing.assert_allclose(I, OL.build_rhs(OL.desc_from_lattice_problem(p), "intensity").reshape(I.shape),
                               rtol=1e-11, atol=1e-14)


def test_cfg5_full_size_linearity_and_direction_shards():
    """BASELINE cfg5 at full size (128^3, 96 directions, 41 nu, moment layout: 516 M unknowns,
    8.25 G intensity DOF) through size-independent properties: linearity, and two direction
    shards (rtk_lattice_partial_moments, summed) reassembling the operator."""
    import torch

    from paper_2602_21958_b200.sharding import LatticeShardedOperator

    p = configs.lattice_config_problem(5)
    gen = torch.Generator(device="cuda").manual_seed(5)
    u = torch.randn(p.n_total, dtype=torch.float64, device="cuda", generator=gen)
    w = torch.randn(p.n_total, dtype=torch.float64, device="cuda", generator=gen)
    au, aw = P.apply_A(p, u), P.apply_A(p, w)
    comb = P.apply_A(p, 2.0 * u - 0.5 * w)
    assert float(torch.linalg.vector_norm(comb - (2.0 * au - 0.5 * aw)) / torch.linalg.vector_norm(comb)) <= 1e-13
    del w, aw, comb
    ops = [LatticeShardedOperator(p, rank=r, world=2, all_reduce=lambda t: t) for r in range(2)]
    m = ops[0].ops.partial_moments(u)
    m += ops[1].ops.partial_moments(u)
    y = ops[0].ops.apply_with_moments(u, m)
    assert float(torch.linalg.vector_norm(y - au) / torch.linalg.vector_norm(au)) <= 1e-12


# Every shipped kernel variant against the oracle (rtk_problem_set_tuning selects it):
# moment layout -- the tiled kernel lattice_mom_tile_kernel (default for IE / exp-linear) with
# 1, 3 and 8 direction groups, and the per-item gather kernel lattice_mom_group_kernel (the
# exp-parabolic path, and IE / exp-linear with lattice_no_tile) with DG = 1, 4 and 8 direction
# groups; intensity layout -- the shared-memory kernel (3D and planar sampling, with and
# without the dt table) and the non-shared-memory fallback lattice_int_kernel.
MOMENT_VARIANTS = [{}, {"lattice_dgz": 1}, {"lattice_dgz": 3}, {"lattice_dgz": 8},
                   {"lattice_no_tile": 1, "lattice_dg": 1}, {"lattice_no_tile": 1, "lattice_dg": 4},
                   {"lattice_no_tile": 1, "lattice_dg": 8}]
INTENSITY_VARIANTS = [{"lattice_no_smem": 1}, {"lattice_no_dtab": 1}, {"lattice_no_planar": 1},
                      {"lattice_no_dtab": 1, "lattice_no_planar": 1}]


def _with_tuning(p, tuning):
    h = p.device()
    for k, v in tuning.items():
        h.set_tuning(k, v)
    return p


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("tuning", MOMENT_VARIANTS, ids=lambda t: ",".join(f"{k}={v}" for k, v in t.items()))
@pytest.mark.parametrize("chars", ["long", "hybrid"])
@pytest.mark.parametrize("fs", ["ie", "exp_linear", "exp_parabolic"])
def test_moment_kernel_variants_match_oracle(case, tuning, chars, fs):
    nx, ny, nz, npol, naz, nf = case
    p = L.lattice_problem(nx, ny, nz, npol, naz, nf, corr_len=2.0, seed=17, layout="moments", formal_solver=fs,
                          characteristics=chars)
    _with_tuning(p, tuning)
    d = OL.desc_from_lattice_problem(p)
    v = np.random.default_rng(nx * 7 + nf).standard_normal(p.n_total)
    assert rel_l2(P.apply_A(p, v), OL.apply_A(d, "moments", v)) <= MATVEC_TOL
    assert rel_l2(P.build_rhs(p), OL.build_rhs(d, "moments")) <= MATVEC_TOL


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("tuning", INTENSITY_VARIANTS, ids=lambda t: ",".join(f"{k}={v}" for k, v in t.items()))
@pytest.mark.parametrize("fs", ["ie", "exp_linear"])
def test_intensity_kernel_variants_match_oracle(case, tuning, fs):
    nx, ny, nz, npol, naz, nf = case
    p = L.lattice_problem(nx, ny, nz, npol, naz, nf, corr_len=2.0, seed=19, layout="intensity", formal_solver=fs)
    _with_tuning(p, tuning)
    d = OL.desc_from_lattice_problem(p)
    v = np.random.default_rng(nx * 5 + nf).standard_normal(p.n_total)
    assert rel_l2(P.apply_A(p, v), OL.apply_A(d, "intensity", v)) <= MATVEC_TOL
    assert rel_l2(P.build_rhs(p), OL.build_rhs(d, "intensity")) <= MATVEC_TOL


def test_fallback_intensity_kernel_rejects_what_it_cannot_do():
    """Without the shared-memory kernel, exp-parabolic and short characteristics in the
    intensity layout are refused (RTK_ERESOURCE -> ResourceLimitError), never approximated."""
    from paper_2602_21958_b200.errors import ResourceLimitError

    for kw in (dict(formal_solver="exp_parabolic"), dict(characteristics="short")):
        p = L.lattice_problem(8, 1, 6, 4, 4, 3, corr_len=1.0, layout="intensity", **kw)
        _with_tuning(p, {"lattice_no_smem": 1})
        with pytest.raises(ResourceLimitError):
            P.apply_A(p, np.ones(p.n_total))


def test_auto_selection_takes_one_direction_group_on_large_steps():
    """A step with > 131,072 (line, frequency-pair) items selects DG = 1 by itself (cfg5's
    path): 64 x 64 lines x 33 pairs; against the oracle with the default tuning."""
    p = L.lattice_problem(64, 64, 4, 4, 2, 66, corr_len=4.0, seed=23, layout="moments")
    _with_tuning(p, {"lattice_no_tile": 1})
    d = OL.desc_from_lattice_problem(p)
    v = np.random.default_rng(23).standard_normal(p.n_total)
    assert rel_l2(P.apply_A(p, v), OL.apply_A(d, "moments", v)) <= MATVEC_TOL


@pytest.mark.parametrize("tuning", [{}, {"lattice_no_tile": 1, "lattice_dg": 1}], ids=["tiled", "group_dg1"])
def test_cfg5_column_geometry_matches_oracle(tuning):
    """BASELINE cfg5 construction at its full depth and angular set (nz = 128, 8 x 12 = 96
    directions, corr 16, eps 1e-5, moment layout) on a 32 x 32 horizontal period with N_nu = 4
    (the oracle takes ~1 min): default selection and cfg5's own kernel instantiation (one
    direction group, lattice_mom_group_kernel<..., 1>) and the tiled kernel."""
    p = configs.lattice_config_problem(5, nx=32, ny=32, n_freq=4)
    _with_tuning(p, tuning)
    d = OL.desc_from_lattice_problem(p)
    v = np.random.default_rng(5).standard_normal(p.n_total)
    assert rel_l2(P.apply_A(p, v), OL.apply_A(d, "moments", v)) <= MATVEC_TOL


def test_cfg5_full_geometry_matches_oracle_fixture():
    """BASELINE cfg5 geometry at FULL size (128^3, 96 directions; N_nu = 4, 805 M intensity DOF)
    against the oracle output committed by tests/golden/make_cfg5_fixture.py (65,536 sampled
    entries and 8 sketches of y = A u; the oracle itself needs ~15 CPU-minutes here).  This
    step size (16,384 lines x 2 pairs) selects the multi-group kernel, so both DG = 1 (cfg5's
    instantiation) and the default are checked."""
    import os

    import torch

    sys_path = os.path.join(os.path.dirname(__file__), "golden")
    z = np.load(os.path.join(sys_path, "cfg5_geometry_nu4.npz"))
    from tests.golden import make_cfg5_fixture as F

    p = configs.lattice_config_problem(5, n_freq=F.N_FREQ)
    assert p.n_total == int(z["n_total"])
    u = np.random.default_rng(F.U_SEED).standard_normal(p.n_total)
    idx = torch.from_numpy(z["index"]).cuda()
    for tuning in ({}, {"lattice_no_tile": 1, "lattice_dg": 1}):
        _with_tuning(p, tuning)
        y = P.apply_A(p, torch.from_numpy(u).cuda())
        ys = y[idx].cpu().numpy()
        assert rel_l2(ys, z["values"]) <= MATVEC_TOL, tuning
        yh = y.cpu().numpy()
        assert abs(np.linalg.norm(yh) - float(z["norm"])) <= 1e-12 * float(z["norm"])
        for r, ref in zip(F.sketch_vectors(p.n_total), z["sketches"]):
            assert abs(r @ yh - ref) <= 1e-11 * float(z["norm"]) * np.sqrt(p.n_total)


@pytest.mark.parametrize("ray", [0, 1])
@pytest.mark.parametrize("tuning", [{}, {"lattice_no_smem": 1}], ids=["smem", "fallback"])
def test_device_transfer_matches_reference_multidim(ray, tuning):
    """The device lattice transfer against the reference's own 2D long characteristics
    (R/multidim.py, tests/golden/make_multidim_golden.py), in the coinciding configuration:
    build_rhs of a one-direction problem whose isotropic thermal source is the golden's
    source for that ray gives Lambda S + the inflow term."""
    from tests import _multidim_golden as MG

    z = MG.load()
    for S, lam in zip(z["source"], z["lambda"]):
        p = MG.column_problem(z, directions=(ray,), thermal=S[..., ray].reshape(-1))
        _with_tuning(p, tuning)
        want = (lam[..., ray] + z["boundary"][..., ray]).reshape(-1)
        assert rel_l2(P.build_rhs(p), want) <= 1e-13
