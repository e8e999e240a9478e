"""Presets, spectrum diagnostics and CLI plumbing on the host (no GPU).

The preset setup arrays are pinned to the reference's own presets through the
golden file (tests/golden/ref_goldens.npz: mono(12, 8), coherent(6, 4, 7),
crd(6, 4, 7) built by R/presets.py); the GPU side of the CLI and the spectrum
is in tests/test_gpu_cli.py.
"""
import json

import numpy as np
import pytest

from paper_2602_21958_b200 import cli, presets, spectrum
from tests import _golden as G

CASES = {"mono": ("mono", 12, 8, 1), "coherent": ("coherent", 6, 4, 7), "crd": ("crd", 6, 4, 7)}


@pytest.mark.parametrize("key", sorted(CASES))
def test_presets_match_reference_setup_arrays(key):
    z = G.load()
    name, ns, nom, nnu = CASES[key]
    p = presets.build(name, n_space=ns, n_angles=nom, n_freq=nnu)
    g = p.grid
    np.testing.assert_array_equal(g.t_nodes, z[f"{key}/t_nodes"])
    np.testing.assert_allclose(g.mu_nodes, z[f"{key}/mu"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(g.angular_weights, z[f"{key}/ang_w"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(g.nu_nodes, z[f"{key}/nu"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(g.frequency_weights, z[f"{key}/freq_w"], rtol=0, atol=1e-14)
    np.testing.assert_allclose(g.profile_values(), z[f"{key}/phi"], rtol=1e-15)
    np.testing.assert_allclose(p.scattering.gamma_table.reshape(z[f"{key}/gamma"].shape), z[f"{key}/gamma"],
                               rtol=1e-14)
    np.testing.assert_array_equal(p.transfer.inflow, z[f"{key}/inflow"])
    np.testing.assert_array_equal(p.thermal, z[f"{key}/thermal"])
    assert type(p.scattering.kernel).__name__ == str(z[f"{key}/kernel"])


def test_aniso2d_and_unknown_presets_are_rejected():
    with pytest.raises(ValueError, match="aniso2d"):
        presets.build("aniso2d", n_space=4, n_angles=4, n_freq=1)
    with pytest.raises(ValueError, match="unknown preset"):
        presets.build("nope", n_space=4, n_angles=4, n_freq=1)


def test_spectrum_of_known_matrix():
    lam = np.array([1.0, 0.9995, 1.0008, 0.5, 2.0, 0.96])
    rep = spectrum.spectrum_of(np.diag(lam), {"preset": "diag"})
    assert rep.n == 6
    assert rep.cluster_fraction == pytest.approx(3 / 6)
    assert rep.cluster_fraction_one_sided == pytest.approx(2 / 6)
    assert rep.min_modulus == pytest.approx(0.5)
    assert rep.outlier_counts == {0.01: 3, 0.05: 2, 0.1: 2, 0.15: 2}
    assert rep.descriptor == {"preset": "diag", "n_total": 6}


def test_clustering_trend():
    mk = lambda counts: spectrum.SpectrumReport(np.ones(2), 1.0, 1.0, 1.0, counts)  # noqa: E731
    ok = spectrum.clustering_trend([mk({0.1: 5}), mk({0.1: 4}), mk({0.1: 6})])
    assert ok.strong_cluster_consistent and ok.outlier_counts == {0.1: [5, 4, 6]}
    bad = spectrum.clustering_trend([mk({0.1: 5}), mk({0.1: 2}), mk({0.1: 5})])
    assert not bad.strong_cluster_consistent
    with pytest.raises(ValueError):
        spectrum.clustering_trend([mk({0.1: 5})])


def test_cli_config_merge_and_errors(tmp_path):
    cfg_file = tmp_path / "c.json"
    cfg_file.write_text(json.dumps({"ns": "7", "tol": 1e-6}))
    args = cli.build_parser().parse_args(["solve", "--config", str(cfg_file), "--tol", "1e-9"])
    cfg = cli.merge_config(args)
    assert cfg["ns"] == "7" and cfg["tol"] == 1e-9 and cfg["preset"] == "mono" and cfg["mode"] == "solve"
    cfg_file.write_text(json.dumps({"bogus": 1}))
    with pytest.raises(cli.ConfigError, match="unknown config keys"):
        cli.merge_config(cli.build_parser().parse_args(["solve", "--config", str(cfg_file)]))
    # invalid configurations exit 1 before any device work (R/cli.py:296-298)
    assert cli.main(["solve", "--preset", "aniso2d", "--out", str(tmp_path / "o")]) == 1
    assert cli.main(["table", "--preset", "aniso2d", "--out", str(tmp_path / "o")]) == 1
    assert cli.main(["solve", "--ns", "4,6", "--out", str(tmp_path / "o")]) == 1
    assert cli.main(["convergence", "--preset", "crd", "--ns", "4,6", "--nnu", "3,5,7",
                     "--out", str(tmp_path / "o")]) == 1
