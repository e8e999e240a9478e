"""Golden fixture for the cfg5-geometry lattice parity test (tests/test_gpu_lattice.py).

The numpy lattice oracle needs ~15 CPU-minutes for one matvec at the full cfg5 geometry
(128^3 grid, 96 directions) even with N_nu reduced to 4, too slow for a test run, so this
script runs it once and stores what the GPU test compares against:
  * 65,536 seeded-random entries of y = A u (index and value),
  * 8 sketches r_k . y with seeded Gaussian r_k, and ||y||.
The input u is regenerated from its seed by the test.  Run from the repo root:
  python tests/golden/make_cfg5_fixture.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import lattice as OL  # noqa: E402
from paper_2602_21958_b200 import configs  # noqa: E402

N_FREQ = 4
U_SEED = 5
N_SAMPLES = 65536
N_SKETCH = 8


def sample_index(n):
    return np.sort(np.random.default_rng(777).choice(n, N_SAMPLES, replace=False))


def sketch_vectors(n):
    rng = np.random.default_rng(778)
    return [rng.standard_normal(n) for _ in range(N_SKETCH)]


def main():
    p = configs.lattice_config_problem(5, n_freq=N_FREQ)
    d = OL.desc_from_lattice_problem(p)
    u = np.random.default_rng(U_SEED).standard_normal(p.n_total)
    y = OL.apply_A(d, "moments", u)
    idx = sample_index(p.n_total)
    sk = np.array([r @ y for r in sketch_vectors(p.n_total)])
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "cfg5_geometry_nu4.npz"), index=idx, values=y[idx],
                        sketches=sk, norm=np.linalg.norm(y), n_total=p.n_total)


if __name__ == "__main__":
    main()
