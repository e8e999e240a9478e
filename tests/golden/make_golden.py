"""Generate golden vectors by running the UNMODIFIED reference (rtkrylov).

Run in the build container only (the reference is not on the GPU box):
    python tests/golden/make_golden.py
Writes tests/golden/ref_goldens.npz.  Every array is produced by the
reference's own public API (R/ = /root/reference/pkg/src/rtkrylov/):
grid/transfer/scattering builders, apply_A, build_rhs, apply_transfer,
apply_scattering, sweep_down/up and gmres.  Inputs are seeded.
Cases that need the (absent) PRD/exp/multi-D physics are not here: the
oracle pins those through reduction identities against these cases.
"""
import os
import sys

sys.dont_write_bytecode = True                    # never write into /root/reference
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rtk_numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import rtkrylov  # noqa: E402
from rtkrylov import presets, _kernels  # noqa: E402
from rtkrylov.grid import Grid  # noqa: E402
from rtkrylov.krylov import SolveConfig, gmres  # noqa: E402
from rtkrylov.operator import RTProblem, apply_A, build_rhs  # noqa: E402
from rtkrylov.quadrature import gauss_legendre, trapezoid  # noqa: E402
from rtkrylov.scattering import CRDKernel, LegendreKernel, apply_scattering, build_scattering  # noqa: E402
from rtkrylov.transfer import apply_transfer, build_transfer  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_goldens.npz")


def gauss(nu):
    nu = np.asarray(nu, dtype=float)
    return np.exp(-nu * nu) / np.sqrt(np.pi)


def log_grid_problem(n_space, n_angles, n_freq, kernel, eps, x_max=5.0, t_lo=-4, t_hi=4):
    """cfg1-shaped problem: log-spaced t, Gaussian profile, thermal eps, zero inflow."""
    t = np.logspace(t_lo, t_hi, n_space)
    dn = gauss_legendre(n_angles // 2, -1.0, 0.0)
    up = gauss_legendre(n_angles // 2, 0.0, 1.0)
    fr = trapezoid(n_freq, -x_max, x_max)
    grid = Grid(t, np.concatenate([dn.nodes, up.nodes]), np.concatenate([dn.weights, up.weights]),
                fr.nodes, fr.weights, gauss)
    transfer = build_transfer(grid, 0.0, 0.0)
    if kernel == "legendre":
        # frequency-flat dipole kernel: conservative when gamma = (1-eps) / (2 sum_f w_f)
        kern = LegendreKernel((1.0, 0.0, 0.5))
        wsum = float(fr.weights.sum())
        gam = lambda tt, mu, nu: (1.0 - eps) / (2.0 * wsum) * np.ones_like(tt + mu + nu)  # noqa: E731
    else:
        kern = CRDKernel(gauss)
        gam = lambda tt, mu, nu: (1.0 - eps) / (2.0 * gauss(nu)) * np.ones_like(tt + mu)  # noqa: E731
    scat = build_scattering(grid, kern, gam)
    return RTProblem(grid, transfer, scat, thermal=np.full(grid.n_total, eps))


def dump_problem(store, key, p, seed, n_vec=2, gmres_cfgs=(), rhs=True):
    g = p.grid
    store[f"{key}/t_nodes"] = g.t_nodes
    store[f"{key}/mu"] = g.mu_nodes
    store[f"{key}/ang_w"] = g.angular_weights
    store[f"{key}/nu"] = g.nu_nodes
    store[f"{key}/freq_w"] = g.frequency_weights
    store[f"{key}/phi"] = np.asarray(g.profile(g.nu_nodes), dtype=float) * np.ones(g.n_freq)
    store[f"{key}/gamma"] = p.scattering.gamma_table
    store[f"{key}/inflow"] = p.transfer.inflow
    store[f"{key}/thermal"] = p.thermal
    store[f"{key}/dtau"] = p.transfer.dtau
    k = p.scattering.kernel
    store[f"{key}/kernel"] = np.array(type(k).__name__)
    if isinstance(k, LegendreKernel):
        store[f"{key}/coefficients"] = np.asarray(k.coefficients)
    rng = np.random.default_rng(seed)
    vs = rng.standard_normal((n_vec, p.n_total))
    store[f"{key}/v"] = vs
    store[f"{key}/Av"] = np.stack([apply_A(p, v) for v in vs])
    store[f"{key}/Sigma_v"] = np.stack([apply_scattering(p.scattering, v) for v in vs])
    store[f"{key}/Lambda_v"] = np.stack([apply_transfer(p.transfer, v) for v in vs])
    if rhs:
        with np.errstate(all="ignore"):
            store[f"{key}/rhs"] = build_rhs(p)
    for name, cfg in gmres_cfgs:
        b = build_rhs(p) if rhs else rng.standard_normal(p.n_total)
        rep = gmres(lambda v: apply_A(p, v), b, cfg)
        store[f"{key}/gmres_{name}/b"] = b
        store[f"{key}/gmres_{name}/solution"] = rep.solution
        store[f"{key}/gmres_{name}/iterations"] = np.array(rep.iterations)
        store[f"{key}/gmres_{name}/history"] = np.asarray(rep.residual_history)
        store[f"{key}/gmres_{name}/converged"] = np.array(rep.converged)
        store[f"{key}/gmres_{name}/true_residual"] = np.array(rep.true_residual)
        store[f"{key}/gmres_{name}/cfg"] = np.array([cfg.rel_tol, cfg.max_iter, -1 if cfg.restart is None else cfg.restart,
                                                       int(cfg.reorthogonalize)], dtype=float)
        print(key, name, "iterations", rep.iterations, "converged", rep.converged, flush=True)


def main():
    store = {}
    store["version"] = np.array(rtkrylov.__version__)
    # --- sweep kernels, the reference unit fixture (T/test_kernels.py:12-16) ---
    rng = np.random.default_rng(0)
    dtau = rng.uniform(0.01, 5.0, size=(7, 19))
    src = rng.standard_normal((7, 20))
    store["sweep/dtau"] = dtau
    store["sweep/src"] = src
    store["sweep/down"] = _kernels.sweep_down(dtau, src)
    store["sweep/up"] = _kernels.sweep_up(dtau, src)
    # --- quadrature ---
    for n in (1, 2, 4, 8, 16, 32):
        q = gauss_legendre(n, 0.0, 1.0)
        store[f"gl/{n}/nodes"] = q.nodes
        store[f"gl/{n}/weights"] = q.weights
    # --- reference presets (T/test_operator.py:20-31) ---
    dump_problem(store, "mono", presets.monochromatic(12, 8), 1,
                 gmres_cfgs=(("full", SolveConfig(rel_tol=1e-10, max_iter=500)),
                             ("r5", SolveConfig(rel_tol=1e-10, max_iter=500, restart=5))))
    dump_problem(store, "coherent", presets.coherent(6, 4, 7), 2,
                 gmres_cfgs=(("full", SolveConfig(rel_tol=1e-12, max_iter=500)),))
    dump_problem(store, "crd", presets.crd(6, 4, 7), 3,
                 gmres_cfgs=(("full", SolveConfig(rel_tol=1e-12, max_iter=500)),))
    # --- cfg1-shaped problems on the reference's own Grid/kernels ---
    dump_problem(store, "log_legendre", log_grid_problem(30, 8, 11, "legendre", 1e-4), 4,
                 gmres_cfgs=(("full", SolveConfig(rel_tol=1e-8, max_iter=2000)),
                             ("r30", SolveConfig(rel_tol=1e-8, max_iter=4000, restart=30))))
    dump_problem(store, "log_crd", log_grid_problem(30, 8, 11, "crd", 1e-4), 5,
                 gmres_cfgs=(("full", SolveConfig(rel_tol=1e-8, max_iter=2000)),))
    # cfg1 geometry exactly (t=logspace(-4,4,100), 8+8 mu, 31 nu on +-5, eps=1e-4) with the
    # reference's frequency-flat dipole LegendreKernel((1,0,1/2)) standing in for dipole x PRD
    dump_problem(store, "cfg1_legendre", log_grid_problem(100, 16, 31, "legendre", 1e-4), 6, n_vec=1,
                 gmres_cfgs=(("full", SolveConfig(rel_tol=1e-8, max_iter=2000)),
                             ("r30", SolveConfig(rel_tol=1e-8, max_iter=6000, restart=30))))
    # cfg1 geometry with the reference's CRDKernel: the hard, slowly converging regime
    dump_problem(store, "cfg1_crd", log_grid_problem(100, 16, 31, "crd", 1e-4), 7, n_vec=1,
                 gmres_cfgs=(("full", SolveConfig(rel_tol=1e-8, max_iter=2000)),
                             ("r30", SolveConfig(rel_tol=1e-8, max_iter=4000, restart=30))))
    np.savez_compressed(OUT, **store)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
