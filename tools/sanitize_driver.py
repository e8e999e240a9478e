"""compute-sanitizer driver: one small launch of every mbarrier / TMA / cluster-DSMEM kernel family
(fused Sigma with a cluster of 2, TMA sweeps of the three formal solvers, the 1D moment-layout
sweep, lattice kernels of both layouts, the CGS2 / MGS passes).  Run as
  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_driver.py
Sizes are small because the sanitizer slows kernels by 10-100x."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import configs  # noqa: E402
from paper_2602_21958_b200 import lattice as L  # noqa: E402

which = sys.argv[1:] or ["fused", "sweeps", "mom1d", "lattice", "krylov"]
gen = torch.Generator(device="cuda").manual_seed(1)


def rnd(n):
    return torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)


if "fused" in which:
    # N_nu = 256 -> clusters of 2 CTAs (DSMEM hand-off), ragged point blocks
    p = configs.slab_problem(2, n_space=37, n_angles=16, n_freq=256)
    y = P.apply_A(p, rnd(p.n_total))
    print("fused", float(y.norm()))
if "sweeps" in which:
    for fs in ("ie", "exp_linear", "exp_parabolic"):
        p = configs.slab_problem(2, n_space=45, n_angles=8, n_freq=128, formal_solver=fs)
        y = P.apply_A(p, rnd(p.n_total))
        b = P.build_rhs(p)
        print("sweep", fs, float(y.norm()))
if "mom1d" in which:
    p = configs.slab_problem(2, n_space=45, n_angles=16, n_freq=128, layout="moments")
    y = P.apply_A(p, rnd(p.n_total))
    print("mom1d", float(y.norm()))
if "lattice" in which:
    for layout in ("intensity", "moments"):
        for fs, ch in (("ie", "long"), ("exp_parabolic", "hybrid")):
            p = L.lattice_problem(8, 6, 7, 4, 4, 6, corr_len=2.0, seed=5, layout=layout, formal_solver=fs,
                                  characteristics=ch)
            y = P.apply_A(p, rnd(p.n_total))
            print("lattice", layout, fs, ch, float(y.norm()))
if "krylov" in which:
    p = configs.slab_problem(1, n_space=30, n_angles=8, n_freq=11)
    b = P.build_rhs(p)
    for orth in (None, "mgs2", "cgs2"):
        for restart in (7, None):
            rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=60, restart=restart, orthogonalization=orth))
            print("gmres", orth, restart, rep.iterations, rep.converged)
    rep = P.bicgstab(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=60))
    print("bicgstab", rep.iterations)
torch.cuda.synchronize()
print("ok")
