"""Golden outputs of the reference's CLI and spectrum module (R/cli.py, R/spectrum.py).

Run in the build container only (the reference is not on the GPU box):
    python tests/golden/make_cli_golden.py
Writes tests/golden/ref_cli.npz by running the UNMODIFIED reference: its
`compute_spectrum` on small presets, and `rtkrylov.cli.main` for the solve,
convergence and table subcommands (outputs read back from the files the CLI
wrote into a temporary directory).
"""
import csv
import json
import os
import sys
import tempfile

sys.dont_write_bytecode = True                    # never write into /root/reference
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rtk_numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from rtkrylov import cli, presets  # noqa: E402
from rtkrylov.spectrum import compute_spectrum  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_cli.npz")

SPECTRA = {"mono_6_4": ("mono", 6, 4, 1), "coherent_4_4_5": ("coherent", 4, 4, 5), "crd_4_4_5": ("crd", 4, 4, 5)}
SOLVES = {
    "solve_crd": ["solve", "--preset", "crd", "--ns", "8", "--nomega", "4", "--nnu", "7", "--tol", "1e-10"],
    "solve_mono_r5": ["solve", "--preset", "mono", "--ns", "12", "--nomega", "8", "--tol", "1e-10", "--restart", "5"],
    "solve_mono_bicg": ["solve", "--preset", "mono", "--ns", "10", "--nomega", "6", "--tol", "1e-10", "--solver",
                        "bicgstab", "--rhs-one"],
}
CONVERGENCE = {"conv_crd": ["convergence", "--preset", "crd", "--ns", "6,10", "--nomega", "4", "--nnu", "5",
                            "--tol", "1e-10"]}
TABLES = {"table_mono": ["table", "--preset", "mono", "--ns", "4,6", "--nomega", "4,6"]}


def read_csv(path):
    with open(path, newline="", encoding="utf-8") as fh:
        rows = list(csv.reader(fh))
    return rows[0], rows[1:]


def main():
    store = {}
    for key, (preset, ns, nom, nnu) in SPECTRA.items():
        rep = compute_spectrum(presets.build(preset, n_space=ns, n_angles=nom, n_freq=nnu))
        store[f"{key}/eigenvalues"] = rep.eigenvalues
        store[f"{key}/cluster_fraction"] = rep.cluster_fraction
        store[f"{key}/cluster_fraction_one_sided"] = rep.cluster_fraction_one_sided
        store[f"{key}/min_modulus"] = rep.min_modulus
        store[f"{key}/outlier_eps"] = np.array(sorted(rep.outlier_counts))
        store[f"{key}/outlier_counts"] = np.array([rep.outlier_counts[e] for e in sorted(rep.outlier_counts)])
    with tempfile.TemporaryDirectory() as tmp:
        for key, argv in SOLVES.items():
            out = os.path.join(tmp, key)
            rc = cli.main(argv + ["--out", out])
            with open(os.path.join(out, "report.json"), encoding="utf-8") as fh:
                rep = json.load(fh)
            header, rows = read_csv(os.path.join(out, "solution.csv"))
            store[f"{key}/argv"] = np.array(argv)
            store[f"{key}/rc"] = rc
            store[f"{key}/iterations"] = rep["iterations"]
            store[f"{key}/converged"] = rep["converged"]
            store[f"{key}/history"] = np.array(rep["residual_history"])
            store[f"{key}/true_residual"] = rep["true_residual"] if rep["true_residual"] is not None else np.nan
            store[f"{key}/header"] = np.array(header)
            store[f"{key}/solution"] = np.array([[float(v) for v in r] for r in rows])
            store[f"{key}/report_keys"] = np.array(sorted(rep))
        for key, argv in CONVERGENCE.items():
            out = os.path.join(tmp, key)
            rc = cli.main(argv + ["--out", out])
            header, rows = read_csv(os.path.join(out, "convergence.csv"))
            store[f"{key}/argv"] = np.array(argv)
            store[f"{key}/rc"] = rc
            store[f"{key}/header"] = np.array(header)
            store[f"{key}/rows"] = np.array(rows)
        for key, argv in TABLES.items():
            out = os.path.join(tmp, key)
            rc = cli.main(argv + ["--out", out])
            header, rows = read_csv(os.path.join(out, "table.csv"))
            store[f"{key}/argv"] = np.array(argv)
            store[f"{key}/rc"] = rc
            store[f"{key}/header"] = np.array(header)
            store[f"{key}/rows"] = np.array(rows)
    np.savez_compressed(OUT, **store)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
