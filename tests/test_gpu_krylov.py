"""Device GMRES / BiCGStab semantics on small dense systems, mirroring the reference's
Krylov unit tests (T/test_krylov.py: GMRES vs LU, n-step termination, monotone history,
true-residual guard, happy breakdown, max_iter, restart = full, zero RHS, BiCGStab) through
the callable path (rtk_gmres / rtk_bicgstab with a C callback, Krylov vectors on the device)."""
import numpy as np
import pytest

import paper_2602_21958_b200 as P
from paper_2602_21958_b200 import configs

pytestmark = pytest.mark.gpu


def _system(n=50, seed=0, shift=4.0):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n)) / np.sqrt(n) + shift * np.eye(n)
    b = rng.standard_normal(n)
    return A, b


def _apply(A):
    return lambda v: A @ np.asarray(v)


def test_gmres_matches_lu():
    A, b = _system()
    rep = P.gmres(_apply(A), b, P.SolveConfig(rel_tol=1e-12, max_iter=200))
    assert rep.converged
    x = np.linalg.solve(A, b)
    assert np.linalg.norm(rep.solution - x) <= 1e-10 * np.linalg.norm(x)


def test_gmres_terminates_in_at_most_n_steps():
    A, b = _system(n=20, shift=0.5, seed=1)
    rep = P.gmres(_apply(A), b, P.SolveConfig(rel_tol=1e-10, max_iter=100))
    assert rep.converged and rep.iterations <= 20


def test_gmres_history_is_monotone_and_true_residual_guarded():
    A, b = _system(seed=2)
    tol = 1e-9
    rep = P.gmres(_apply(A), b, P.SolveConfig(rel_tol=tol, max_iter=200))
    h = np.asarray(rep.residual_history)
    assert np.all(np.diff(h) <= 1e-14)
    true = np.linalg.norm(b - A @ rep.solution) / np.linalg.norm(b)
    assert rep.converged and true <= 10 * tol
    assert abs(rep.true_residual - true) <= 1e-12


def test_gmres_happy_breakdown_on_an_invariant_subspace():
    n = 30
    A = np.diag(np.arange(1.0, n + 1))
    b = np.zeros(n)
    b[3] = 2.0                                           # an eigenvector: Krylov space of dimension 1
    rep = P.gmres(_apply(A), b, P.SolveConfig(rel_tol=1e-12, max_iter=50))
    assert rep.converged and rep.iterations == 1
    np.testing.assert_allclose(rep.solution, np.linalg.solve(A, b), rtol=1e-13, atol=1e-15)


def test_gmres_stops_at_max_iter():
    A, b = _system(shift=0.2, seed=3)
    rep = P.gmres(_apply(A), b, P.SolveConfig(rel_tol=1e-14, max_iter=5))
    assert not rep.converged and rep.iterations == 5 and len(rep.residual_history) == 5


def test_gmres_restart_larger_than_the_solve_equals_full_gmres():
    A, b = _system(seed=4)
    full = P.gmres(_apply(A), b, P.SolveConfig(rel_tol=1e-10, max_iter=200))
    rst = P.gmres(_apply(A), b, P.SolveConfig(rel_tol=1e-10, max_iter=200, restart=full.iterations + 5))
    assert rst.iterations == full.iterations
    np.testing.assert_array_equal(rst.residual_history, full.residual_history)
    np.testing.assert_array_equal(rst.solution, full.solution)


def test_zero_rhs_returns_the_trivial_report():
    A, _ = _system()
    for solve, cfg in ((P.gmres, P.SolveConfig()), (P.bicgstab, P.SolveConfig(method="bicgstab"))):
        rep = solve(_apply(A), np.zeros(50), cfg)
        assert rep.converged and rep.iterations == 0 and list(rep.residual_history) == [0.0]
        assert not np.any(rep.solution)


def test_bicgstab_matches_lu():
    A, b = _system(seed=5)
    rep = P.bicgstab(_apply(A), b, P.SolveConfig(method="bicgstab", rel_tol=1e-12, max_iter=200))
    assert rep.converged
    x = np.linalg.solve(A, b)
    assert np.linalg.norm(rep.solution - x) <= 1e-9 * np.linalg.norm(x)


def test_bicgstab_within_twice_gmres_iterations_on_a_preset():
    """T/test_krylov.py:150-162: on a reference preset BiCGStab needs at most twice the GMRES count."""
    from paper_2602_21958_b200 import presets

    p = presets.build("crd", n_space=60, n_angles=8, n_freq=9)
    b = P.build_rhs(p)
    g = P.gmres(p, b, P.SolveConfig(rel_tol=1e-10, max_iter=500))
    s = P.bicgstab(P.operator(p), b, P.SolveConfig(method="bicgstab", rel_tol=1e-10, max_iter=500))
    assert g.converged and s.converged and s.iterations <= 2 * g.iterations


def test_solve_config_validation():
    with pytest.raises(ValueError):
        P.SolveConfig(rel_tol=0.0)
    with pytest.raises(ValueError):
        P.SolveConfig(max_iter=0)
    with pytest.raises(ValueError):
        P.SolveConfig(restart=0)


def test_device_tensor_rhs_through_the_callable_path():
    import torch

    A, b = _system(seed=6)
    At = torch.from_numpy(A).cuda()
    rep = P.gmres(lambda v: At @ v, torch.from_numpy(b).cuda(), P.SolveConfig(rel_tol=1e-12, max_iter=200))
    assert rep.converged and rep.solution.is_cuda
    x = np.linalg.solve(A, b)
    assert np.linalg.norm(rep.solution.cpu().numpy() - x) <= 1e-10 * np.linalg.norm(x)
