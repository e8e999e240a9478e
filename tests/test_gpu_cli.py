"""The B200 CLI and spectrum against the reference CLI / spectrum outputs.

Goldens: tests/golden/ref_cli.npz, written by tests/golden/make_cli_golden.py
running the unmodified reference (`rtkrylov.cli.main`, `compute_spectrum`).
Tolerances: eigenvalues matched to 1e-9 absolute (materialised by device
matvecs, LAPACK on the host as in the reference); solve iteration counts
within +-1 (equal in practice), residual-history prefix 1e-8 relative and
solutions 1e-7 relative (BASELINE north_star).
"""
import csv
import json
import os

import numpy as np
import pytest

from paper_2602_21958_b200 import cli, presets
from paper_2602_21958_b200.spectrum import compute_spectrum

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_cli.npz")
SPECTRA = {"mono_6_4": ("mono", 6, 4, 1), "coherent_4_4_5": ("coherent", 4, 4, 5), "crd_4_4_5": ("crd", 4, 4, 5)}


@pytest.fixture(scope="module")
def z():
    f = np.load(GOLD)
    return {k: f[k] for k in f.files}


def _read_csv(path):
    with open(path, newline="", encoding="utf-8") as fh:
        rows = list(csv.reader(fh))
    return rows[0], rows[1:]


@pytest.mark.parametrize("key", sorted(SPECTRA))
def test_spectrum_matches_reference(z, key):
    name, ns, nom, nnu = SPECTRA[key]
    rep = compute_spectrum(presets.build(name, n_space=ns, n_angles=nom, n_freq=nnu))
    ref = z[f"{key}/eigenvalues"]
    assert rep.n == ref.size
    # each reference eigenvalue has a device-materialised counterpart (multiset match)
    ours = list(rep.eigenvalues)
    for lam in ref:
        i = int(np.argmin([abs(lam - o) for o in ours]))
        assert abs(lam - ours[i]) <= 1e-9
        ours.pop(i)
    assert rep.cluster_fraction == pytest.approx(float(z[f"{key}/cluster_fraction"]), abs=1e-15)
    assert rep.cluster_fraction_one_sided == pytest.approx(float(z[f"{key}/cluster_fraction_one_sided"]), abs=1e-15)
    assert rep.min_modulus == pytest.approx(float(z[f"{key}/min_modulus"]), abs=1e-10)
    eps = z[f"{key}/outlier_eps"]
    assert [rep.outlier_counts[float(e)] for e in eps] == list(z[f"{key}/outlier_counts"])


@pytest.mark.parametrize("key", ["solve_crd", "solve_mono_r5", "solve_mono_bicg"])
def test_cli_solve_matches_reference_cli(z, key, tmp_path):
    argv = [str(a) for a in z[f"{key}/argv"]]
    rc = cli.main(argv + ["--out", str(tmp_path)])
    assert rc == int(z[f"{key}/rc"])
    with open(tmp_path / "report.json", encoding="utf-8") as fh:
        rep = json.load(fh)
    assert sorted(rep) == list(z[f"{key}/report_keys"])
    assert rep["schema_version"] == 1 and rep["kind"] == "solve"
    assert abs(rep["iterations"] - int(z[f"{key}/iterations"])) <= 1
    assert rep["converged"] == bool(z[f"{key}/converged"])
    hist, ref_hist = np.array(rep["residual_history"]), z[f"{key}/history"]
    k = min(hist.size, ref_hist.size) - 1
    np.testing.assert_allclose(hist[:k], ref_hist[:k], rtol=1e-8, atol=1e-13)
    header, rows = _read_csv(tmp_path / "solution.csv")
    assert header == list(z[f"{key}/header"])
    sol = np.array([[float(v) for v in r] for r in rows])
    ref = z[f"{key}/solution"]
    np.testing.assert_array_equal(sol[:, :3], ref[:, :3])          # t, mu, nu columns written identically
    assert np.linalg.norm(sol[:, 3] - ref[:, 3]) <= 1e-7 * np.linalg.norm(ref[:, 3])


def test_cli_convergence_matches_reference_cli(z, tmp_path):
    argv = [str(a) for a in z["conv_crd/argv"]]
    assert cli.main(argv + ["--out", str(tmp_path)]) == int(z["conv_crd/rc"])
    header, rows = _read_csv(tmp_path / "convergence.csv")
    assert header == list(z["conv_crd/header"])
    ref = z["conv_crd/rows"]

    def runs(table):
        out = {}
        for size, method, it, res, conv in table:
            out.setdefault((size, method), []).append((int(it), float(res), conv))
        return out

    ours, theirs = runs(rows), runs(ref)
    assert sorted(ours) == sorted(theirs)
    for key, seq in theirs.items():
        mine = ours[key]
        assert abs(len(mine) - len(seq)) <= 1
        assert mine[0][2] == seq[0][2]
        k = min(len(mine), len(seq)) - 1
        np.testing.assert_allclose([r for _, r, _ in mine[:k]], [r for _, r, _ in seq[:k]], rtol=1e-8, atol=1e-13)


def test_cli_table_matches_reference_cli(z, tmp_path):
    argv = [str(a) for a in z["table_mono/argv"]]
    assert cli.main(argv + ["--out", str(tmp_path)]) == int(z["table_mono/rc"])
    header, rows = _read_csv(tmp_path / "table.csv")
    assert header == list(z["table_mono/header"])
    ref = z["table_mono/rows"]
    assert len(rows) == len(ref)
    for r, q in zip(rows, ref):
        assert r[:4] == list(q[:4])
        assert float(r[4]) == float(q[4]) and float(r[5]) == float(q[5])
        assert abs(float(r[6]) - float(q[6])) <= 1e-10
