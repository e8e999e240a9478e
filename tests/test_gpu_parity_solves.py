"""GMRES to 1e-8 on reduced BASELINE configurations, device vs the CPU oracle (north star:
iteration count within +-1, converged solution within 1e-7).

The oracle solves (tests/golden/make_reduced_gmres.py: the reference's MGS GMRES control
flow on the oracle operators, 8-35 CPU-minutes each) are committed as fixtures; the device
solves run here in seconds.  Unrestarted, so the +-1 bound applies (restarted counts have
the reference's own noise band, tests/test_gpu_slab.py::iteration_band).
"""
import os

import numpy as np
import pytest

import paper_2602_21958_b200 as P
from tests._problems import rel_l2

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["cfg2r_intensity", "cfg2r_moments", "cfg3r_moments", "cfg4r_moments", "cfg5r_moments"]


def _fixture(case):
    return np.load(os.path.join(GOLDEN, f"reduced_gmres_{case}.npz"))


def _product_problem(case):
    from paper_2602_21958_b200 import configs

    if case.startswith("cfg2r"):
        return configs.slab_problem(2, n_space=300, n_angles=16, n_freq=64, layout=case.split("_")[1])
    cfg = int(case[3])
    kw = dict(nx=64, ny=1, nz=64) if cfg == 3 else dict(nx=16, ny=16, nz=16)
    return configs.lattice_config_problem(cfg, layout="moments", **kw)


def _check_solution(x, z):
    """Full solution, or the fixture's sampled entries, norm and sketches (large cases)."""
    if "solution" in z:
        assert rel_l2(x, z["solution"]) <= 1e-7
        return
    from tests.golden import make_reduced_gmres as M

    norm = float(z["norm"])
    assert rel_l2(x[z["index"]], z["values"]) <= 1e-7
    assert abs(np.linalg.norm(x) - norm) <= 1e-7 * norm
    for r, s in zip(M.sketch_vectors(x.size), z["sketches"]):
        assert abs(r @ x - s) <= 1e-7 * norm * np.sqrt(x.size)


@pytest.mark.parametrize("orth", [None, "cgs2"], ids=["reference_mgs", "cgs2"])
@pytest.mark.parametrize("case", CASES)
def test_reduced_config_gmres_to_1e8_matches_oracle(case, orth):
    z = _fixture(case)
    p = _product_problem(case)
    assert p.n_total == int(z["n_total"])
    b = P.build_rhs(p)
    rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=3000, orthogonalization=orth))
    assert rep.converged and bool(z["converged"])
    assert abs(rep.iterations - int(z["iterations"])) <= 1, (rep.iterations, int(z["iterations"]))
    k = min(len(rep.residual_history), len(z["history"]), 100)
    np.testing.assert_allclose(rep.residual_history[:k], z["history"][:k], rtol=1e-9, atol=1e-14)
    assert rep.true_residual <= 1e-7
    _check_solution(np.asarray(rep.solution), z)
