"""Golden GMRES-to-1e-8 solves of reduced BASELINE configurations by the CPU oracle.

The oracle (oracle/rt_oracle.py gmres: the reference's MGS control flow, R/krylov.py:56-158,
pinned to the reference's own GMRES goldens; operators oracle/rt_oracle.py and
oracle/lattice.py) needs 8-35 CPU-minutes per solve here, too slow for a test run, so this
script runs each solve once and stores what tests/test_gpu_parity_solves.py compares against:
iterations, converged flag, the residual history, and the solution -- in full when it has at
most 50,000 entries, otherwise 65,536 seeded sampled entries + its norm + 8 seeded sketches.

Cases (VERDICT r1 "next round" 2), all unrestarted, rel_tol 1e-8:
  cfg2r_intensity / cfg2r_moments  cfg2 construction at N_z = 300, 16 mu, 64 nu (tau to 1e6, eps 1e-6)
  cfg3r_moments                    cfg3 construction on a 64 x 64 2D slab (8 x 16 directions, 41 nu)
  cfg4r_moments                    cfg4 construction on 16^3 (8 x 16 directions, 31 nu)
  cfg5r_moments                    cfg5 construction on 16^3 (8 x 12 directions, 41 nu, eps 1e-5)
Run from the repo root:  python tests/golden/make_reduced_gmres.py [case ...]
Writes tests/golden/reduced_gmres_<case>.npz.
"""
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

FULL_MAX = 50000
N_SAMPLES = 65536
N_SKETCH = 8
REL_TOL = 1e-8


def build(case):
    """(product problem, oracle apply, oracle rhs) of a case."""
    from oracle import lattice as OL
    from oracle import rt_oracle as ro
    from paper_2602_21958_b200 import configs

    if case.startswith("cfg2r"):
        layout = case.split("_")[1]
        p = configs.slab_problem(2, n_space=300, n_angles=16, n_freq=64, layout=layout)
        d = ro.desc_from_problem(p)
        if layout == "moments":
            return p, (lambda v: ro.apply_A_moments(d, v)), ro.build_rhs_moments(d)
        return p, (lambda v: ro.apply_A(d, v)), ro.build_rhs(d)
    cfg = int(case[3])
    kw = dict(nx=64, ny=1, nz=64) if cfg == 3 else dict(nx=16, ny=16, nz=16)
    p = configs.lattice_config_problem(cfg, layout="moments", **kw)
    d = OL.desc_from_lattice_problem(p)
    return p, (lambda v: OL.apply_A(d, "moments", v)), OL.build_rhs(d, "moments")


def sample_index(n):
    return np.sort(np.random.default_rng(901).choice(n, min(n, N_SAMPLES), replace=False))


def sketch_vectors(n):
    rng = np.random.default_rng(902)
    return [rng.standard_normal(n) for _ in range(N_SKETCH)]


def path(case):
    return os.path.join(ROOT, "tests", "golden", f"reduced_gmres_{case}.npz")


def run(case):
    from oracle import rt_oracle as ro

    t0 = time.time()
    p, apply, b = build(case)
    rep = ro.gmres(apply, b, rel_tol=REL_TOL, max_iter=3000)
    x = np.asarray(rep.solution)
    out = dict(iterations=rep.iterations, converged=rep.converged, history=np.asarray(rep.residual_history),
               true_residual=rep.true_residual, n_total=x.size, norm=np.linalg.norm(x))
    if x.size <= FULL_MAX:
        out["solution"] = x
    else:
        idx = sample_index(x.size)
        out["index"] = idx
        out["values"] = x[idx]
        out["sketches"] = np.array([r @ x for r in sketch_vectors(x.size)])
    np.savez_compressed(path(case), **out)
    print(case, rep.iterations, rep.converged, f"{time.time() - t0:.0f} s", flush=True)


CASES = ["cfg2r_intensity", "cfg2r_moments", "cfg3r_moments", "cfg4r_moments", "cfg5r_moments"]

if __name__ == "__main__":
    todo = sys.argv[1:] or CASES
    with mp.get_context("spawn").Pool(len(todo)) as pool:
        pool.map(run, todo)
