"""Seeded synthetic stand-ins for the BASELINE configurations (host-side setup).

BASELINE.json names five configurations; the paper's 3D atmosphere is not
available, so seeded synthetic inputs with the stated shapes stand in for
it (DESIGN.md "Configurations" records every choice the BASELINE text
leaves open).  Seeds: numpy default_rng(21958 + cfg).
"""

from __future__ import annotations

import numpy as np

from paper_2602_21958_b200.grid import grid_from_nodes
from paper_2602_21958_b200.operator import RTProblem
from paper_2602_21958_b200.redistribution import gaussian_profile, prd_matrix
from paper_2602_21958_b200.scattering import DipolePRDKernel, build_scattering
from paper_2602_21958_b200.transfer import build_transfer

SEED_BASE = 21958
PRD_COHERENCE = 0.5
DIPOLE = (1.0, 0.0, 0.5)

SLAB_CONFIGS = {
    # cfg: (n_space, n_angles, n_freq, x_max, eps, log10 t range, lognormal sigma, restart)
    1: dict(n_space=100, n_angles=16, n_freq=31, x_max=5.0, eps=1e-4, t_range=(-4.0, 4.0), sigma=0.0, restart=30),
    2: dict(n_space=2000, n_angles=64, n_freq=512, x_max=8.0, eps=1e-6, t_range=(-6.0, 6.0), sigma=0.3, restart=30),
}


def slab_t_nodes(n_space: int, t_range, sigma: float, seed: int) -> np.ndarray:
    """Log-spaced frequency-integrated optical depth; optionally the increments
    (kappa * dz) get a seeded log-normal factor exp(sigma xi - sigma^2/2)."""
    base = np.logspace(t_range[0], t_range[1], n_space)
    if sigma == 0.0:
        return base
    rng = np.random.default_rng(seed)
    dt = np.diff(base) * np.exp(sigma * rng.standard_normal(n_space - 1) - 0.5 * sigma * sigma)
    return np.concatenate([[base[0]], base[0] + np.cumsum(dt)])


def slab_problem(cfg: int = 1, formal_solver: str = "ie", n_space: int = None, n_angles: int = None,
                 n_freq: int = None, coherence: float = PRD_COHERENCE, kernel=None,
                 layout: str = "intensity") -> RTProblem:
    """1D slab with dipole x PRD scattering, Planck B = 1, zero incident intensity.

    gamma = (1 - eps) / (2 phi) (s_d = 2 in 1D), thermal = eps B; R is the
    discretely normalised PRD matrix of redistribution.prd_matrix.
    Overrides of n_space / n_angles / n_freq give reduced parity cases of the
    same construction.
    """
    c = dict(SLAB_CONFIGS[cfg])
    if n_space is not None:
        c["n_space"] = n_space
    if n_angles is not None:
        c["n_angles"] = n_angles
    if n_freq is not None:
        c["n_freq"] = n_freq
    eps = c["eps"]
    t = slab_t_nodes(c["n_space"], c["t_range"], c["sigma"], SEED_BASE + cfg)
    grid = grid_from_nodes(t, c["n_angles"], c["n_freq"], -c["x_max"], c["x_max"], gaussian_profile)
    phi = grid.profile_values()
    if kernel is None:
        R = prd_matrix(grid.nu_nodes, grid.frequency_weights, phi, coherence)
        kernel = DipolePRDKernel(R, DIPOLE)
    transfer = build_transfer(grid, 0.0, 0.0, formal_solver=formal_solver)

    def gamma(tt, mu, nu):
        return (1.0 - eps) / (2.0 * gaussian_profile(nu)) * np.ones_like(tt + mu)

    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        scattering = build_scattering(grid, kernel, gamma)
    return RTProblem(grid=grid, transfer=transfer, scattering=scattering, thermal=np.full(grid.n_total, eps),
                     layout=layout,
                     descriptor=dict(config=cfg, formal_solver=formal_solver, eps=eps, coherence=coherence,
                                     restart=c["restart"], **{k: c[k] for k in ("n_space", "n_angles", "n_freq")}))


def config_summary(cfg: int) -> dict:
    c = SLAB_CONFIGS[cfg]
    n = c["n_space"] * c["n_angles"] * c["n_freq"]
    return dict(cfg=cfg, n_dof=n, vector_bytes=8 * n, **c)


def dof(cfg: int) -> int:
    c = SLAB_CONFIGS[cfg]
    return c["n_space"] * c["n_angles"] * c["n_freq"]


# Multi-D configurations 3-5 on the periodic lattice: grid, angular set
# (n_polar x n_azimuth directions), N_nu, opacity correlation length (cells), eps, the unknown
# layout the configuration is run in (cfg4/5: moment layout -- an intensity vector would be
# 8-66 GB) and the GMRES restart (BASELINE: 20 for cfg5; None = unrestarted).
LATTICE_CONFIGS = {
    3: dict(nx=256, ny=1, nz=256, n_polar=8, n_azimuth=16, n_freq=41, corr_len=16.0, eps=1e-4, layout="intensity"),
    4: dict(nx=64, ny=64, nz=64, n_polar=8, n_azimuth=16, n_freq=31, corr_len=8.0, eps=1e-4, layout="moments"),
    5: dict(nx=128, ny=128, nz=128, n_polar=8, n_azimuth=12, n_freq=41, corr_len=16.0, eps=1e-5, layout="moments"),
}
LATTICE_RESTART = {3: 40, 4: None, 5: 20}


def lattice_config_problem(cfg: int, **overrides):
    """BASELINE configuration 3, 4 or 5 (seed 21958 + cfg); keyword overrides give reduced
    parity cases of the same construction (e.g. nx=ny=nz=16, or another layout)."""
    from paper_2602_21958_b200.lattice import lattice_problem

    kw = dict(LATTICE_CONFIGS[cfg])
    kw.update(overrides)
    return lattice_problem(seed=SEED_BASE + cfg, **kw)
