"""Golden vectors from the reference's OWN 2D long-characteristics code (R/multidim.py), on a
configuration where it and this build's periodic-lattice long characteristics coincide.

Run in the build container only (the reference is not on the GPU box):
    python tests/golden/make_multidim_golden.py
Writes tests/golden/ref_multidim.npz.

Coinciding configuration: a CartesianGrid2D rectangle with unit
spacing hx = hy = 1 (R/multidim.py:41-76) and the two directions along its y axis, d = (0, +1)
and (0, -1) -- set on grid.directions before build_transfer_2d, which traces whatever
directions the grid holds (R/multidim.py:334-336).  Then
  * trace_rays seeds one line per bottom (top) edge node and puts its nodes on the grid
    nodes (arc step 1, R/multidim.py:141-177), so the bilinear Cartesian->line map and the
    inverse-distance line->Cartesian map are both selections (R/multidim.py:201-267);
  * the opacity chi(x, y) = a(x) (1 + 0.3 y) is linear along each line, so the reference's
    midpoint optical depth (R/multidim.py:341-343) equals the lattice's trapezoid one;
  * the line recursion is the reference's IE sweep (R/_kernels.py sweep_lines).
On the lattice this is the 2D slab nx = n_x, ny = 1, nz = n_y with the vertical directions
Omega = (0, 0, +-1), reference y_j = lattice layer k = nz - 1 - j, reference d = (0, +1)
(upward) = lattice Omega_z > 0 (enters at the bottom layer).
Stored: the reference's homogeneous transfer of seeded per-ray sources
(TransferOperator2D.apply_space_major), its boundary term for constant inflows
(boundary_space_major), and the lattice-order inputs.
"""
import os
import sys

sys.dont_write_bytecode = True                    # never write into /root/reference
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rtk_numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from rtkrylov.multidim import CartesianGrid2D, build_transfer_2d  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_multidim.npz")
N_X, N_Y = 7, 11
INFLOW_BOTTOM, INFLOW_TOP = 1.0, 0.25


def column_opacity():
    return np.random.default_rng(2602).uniform(0.2, 3.0, N_X)


def chi_fn(x, y):
    a = column_opacity()
    return a[np.rint(np.asarray(x)).astype(int)] * (1.0 + 0.3 * np.asarray(y))


def inflow_fn(x, y):
    return INFLOW_BOTTOM if y == 0.0 else INFLOW_TOP


def ref_to_lattice(v_ref):
    """Reference (ix * n_y + iy, ray k) -> lattice (layer, column, direction) order."""
    v = v_ref.reshape(N_X, N_Y, 2)
    return np.ascontiguousarray(v[:, ::-1, :].transpose(1, 0, 2))   # [k = N_Y-1-iy][ix][ray]


def main():
    grid = CartesianGrid2D(N_X, N_Y, 2, domain=(0.0, N_X - 1.0, 0.0, N_Y - 1.0))
    grid.directions = np.array([[0.0, 1.0], [0.0, -1.0]])
    tr = build_transfer_2d(grid, chi=chi_fn, inflow=inflow_fn)
    rng = np.random.default_rng(21958)
    srcs = rng.uniform(0.0, 2.0, (3, grid.n_total))
    out = {"source": np.stack([ref_to_lattice(s) for s in srcs]),
           "lambda": np.stack([ref_to_lattice(tr.apply_space_major(s)) for s in srcs]),
           "boundary": ref_to_lattice(tr.boundary_space_major()),
           "column_opacity": column_opacity(), "n_x": N_X, "n_y": N_Y,
           "inflow_bottom": INFLOW_BOTTOM, "inflow_top": INFLOW_TOP}
    np.savez(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
