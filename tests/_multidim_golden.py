"""Lattice problems for the reference-multidim coinciding configuration
(tests/golden/make_multidim_golden.py): a 2D slab with the vertical directions only."""
import os

import numpy as np

from paper_2602_21958_b200 import lattice as L

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_multidim.npz")


def load():
    return np.load(PATH)


def lattice_chi(z):
    """chi at lattice nodes s = k * nx + i: a(x_i) (1 + 0.3 y) with y = nz - 1 - k."""
    nx, nz = int(z["n_x"]), int(z["n_y"])
    a = z["column_opacity"]
    y = (nz - 1 - np.arange(nz))[:, None]
    return (a[None, :] * (1.0 + 0.3 * y)).reshape(-1)


def column_problem(z, directions=(0, 1), thermal=None):
    """LatticeProblem on the golden's grid with the reference's rays `directions` (0: d = (0, +1)
    = Omega_z > 0, 1: d = (0, -1)); one frequency with phi = 1, no scattering."""
    nx, nz = int(z["n_x"]), int(z["n_y"])
    omega = np.array([[0.0, 0.0, 1.0], [0.0, 0.0, -1.0]])[list(directions)]
    nd = omega.shape[0]
    n_space = nx * nz
    th = np.zeros((n_space, 1)) if thermal is None else np.asarray(thermal, dtype=float).reshape(n_space, 1)
    return L.LatticeProblem(nx=nx, ny=1, nz=nz, omega=omega, dir_w=np.full(nd, 2 * np.pi), nu=np.zeros(1),
                            freq_w=np.ones(1), phi=np.ones(1), ybasis=np.ones((1, nd)), coeffs=np.ones(1),
                            R=np.ones((1, 1)), gamma=np.zeros((n_space, 1)), chi=lattice_chi(z), thermal=th,
                            inflow_top=np.full(1, float(z["inflow_top"])),
                            inflow_bottom=np.full(1, float(z["inflow_bottom"])), layout="intensity")
