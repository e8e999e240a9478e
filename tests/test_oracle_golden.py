"""Pin the CPU oracle against vectors produced by the unmodified reference (CPU only)."""
import numpy as np
import pytest

from oracle import rt_oracle as ro
from tests import _golden as G


def test_sweeps_match_reference_fixture():
    z = G.load()
    # T/test_kernels.py:19-26 fixture, reference numba output
    np.testing.assert_array_equal(ro.sweep_down(z["sweep/dtau"], z["sweep/src"]), z["sweep/down"])
    np.testing.assert_array_equal(ro.sweep_up(z["sweep/dtau"], z["sweep/src"]), z["sweep/up"])


@pytest.mark.parametrize("n", [1, 2, 4, 8, 16, 32])
def test_gauss_legendre_matches_reference(n):
    z = G.load()
    x, w = ro.gauss_legendre(n, 0.0, 1.0)
    np.testing.assert_array_equal(x, z[f"gl/{n}/nodes"])
    np.testing.assert_array_equal(w, z[f"gl/{n}/weights"])


@pytest.mark.parametrize("key", G.CASES)
def test_delta_tau_table_matches_reference(key):
    d = G.desc(key)
    np.testing.assert_array_equal(ro.delta_tau_table(d), G.load()[f"{key}/dtau"])


@pytest.mark.parametrize("key", G.CASES)
def test_operator_pieces_match_reference(key):
    z = G.load()
    d = G.desc(key)
    for v, sv, lv, av in zip(z[f"{key}/v"], z[f"{key}/Sigma_v"], z[f"{key}/Lambda_v"], z[f"{key}/Av"]):
        np.testing.assert_allclose(ro.apply_sigma(d, v), sv, rtol=1e-12, atol=1e-12 * np.abs(sv).max())
        np.testing.assert_array_equal(ro.apply_transfer(d, v), lv)
        av_o = ro.apply_A(d, v)
        assert np.linalg.norm(av_o - av) <= 1e-13 * np.linalg.norm(av)


@pytest.mark.parametrize("key", G.CASES)
def test_rhs_matches_reference(key):
    z = G.load()
    d = G.desc(key)
    ref = z[f"{key}/rhs"]
    ours = ro.build_rhs(d)
    np.testing.assert_allclose(ours, ref, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("key", ["mono", "coherent", "crd", "log_legendre", "log_crd", "cfg1_legendre", "cfg1_crd"])
def test_gmres_matches_reference(key):
    d = G.desc(key)
    for case in G.gmres_cases(key):
        if case["name"] == "gmres_r30" and key == "cfg1_crd":
            continue  # long; covered by the slow test below
        rep = ro.gmres(lambda v: ro.apply_A(d, v), case["b"], rel_tol=case["rel_tol"], max_iter=case["max_iter"],
                       restart=case["restart"], reorthogonalize=case["reorthogonalize"])
        assert rep.converged == case["converged"]
        assert abs(rep.iterations - case["iterations"]) <= 1
        k = min(len(rep.residual_history), len(case["history"]), 30)
        np.testing.assert_allclose(rep.residual_history[:k], case["history"][:k], rtol=1e-9, atol=1e-13)
        ref = case["solution"]
        assert np.linalg.norm(rep.solution - ref) <= 1e-7 * np.linalg.norm(ref)


@pytest.mark.slow
def test_gmres_restart30_cfg1_crd_matches_reference():
    d = G.desc("cfg1_crd")
    case = [c for c in G.gmres_cases("cfg1_crd") if c["name"] == "gmres_r30"][0]
    rep = ro.gmres(lambda v: ro.apply_A(d, v), case["b"], rel_tol=case["rel_tol"], max_iter=case["max_iter"],
                   restart=case["restart"])
    assert rep.converged and abs(rep.iterations - case["iterations"]) <= 15
    np.testing.assert_allclose(rep.residual_history[:100], case["history"][:100], rtol=1e-9, atol=1e-13)
