"""The reference's OWN iteration-count noise band for restarted GMRES.

Restarted GMRES on a slowly converging problem amplifies last-bit differences: the
unmodified reference (rtkrylov, run here) needs a different number of iterations when its
right-hand side is perturbed by one ulp.  For every restarted golden case of
tests/golden/ref_goldens.npz this script re-runs the reference's gmres (same problem, same
SolveConfig) on 16 ulp-perturbed copies b (1 + 2.2e-16 xi) and stores the min / max
iteration count.  tests/test_gpu_slab.py accepts a device count inside
[min - 1, max + 1]: the reference's own band plus the north star's +-1.

Run in the build container only:  python tests/golden/make_gmres_bands.py
Writes tests/golden/ref_gmres_bands.npz.
"""
import os
import sys

sys.dont_write_bytecode = True
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rtk_numba_cache")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

import make_golden as MG  # noqa: E402  (puts /root/reference/pkg/src on sys.path)
from rtkrylov import presets  # noqa: E402
from rtkrylov.krylov import SolveConfig, gmres  # noqa: E402
from rtkrylov.operator import apply_A  # noqa: E402

OUT = os.path.join(HERE, "ref_gmres_bands.npz")
N_PERTURB = 16

# the restarted golden cases (make_golden.main), rebuilt with the same reference constructors
CASES = {
    "mono/gmres_r5": (lambda: presets.monochromatic(12, 8), SolveConfig(rel_tol=1e-10, max_iter=500, restart=5)),
    "log_legendre/gmres_r30": (lambda: MG.log_grid_problem(30, 8, 11, "legendre", 1e-4),
                               SolveConfig(rel_tol=1e-8, max_iter=4000, restart=30)),
    "cfg1_legendre/gmres_r30": (lambda: MG.log_grid_problem(100, 16, 31, "legendre", 1e-4),
                                SolveConfig(rel_tol=1e-8, max_iter=6000, restart=30)),
    "cfg1_crd/gmres_r30": (lambda: MG.log_grid_problem(100, 16, 31, "crd", 1e-4),
                           SolveConfig(rel_tol=1e-8, max_iter=4000, restart=30)),
}


def main():
    gold = np.load(MG.OUT)
    store = {}
    for key, (build, cfg) in CASES.items():
        p = build()
        b = gold[f"{key}/b"]
        its = []
        for s in range(N_PERTURB):
            xi = np.random.default_rng(s).standard_normal(b.size)
            rep = gmres(lambda v: apply_A(p, v), b * (1.0 + 2.2e-16 * xi), cfg)
            its.append(rep.iterations)
        store[f"{key}/iterations"] = np.array(its)
        print(key, "golden", int(gold[f"{key}/iterations"]), "perturbed", sorted(its), flush=True)
    np.savez(OUT, **store)


if __name__ == "__main__":
    main()
