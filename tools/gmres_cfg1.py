"""Time cfg1 GMRES to 1e-8 (restart 30 and unrestarted), best of 5 (development tool)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2602_21958_b200 as P  # noqa: E402
from paper_2602_21958_b200 import configs  # noqa: E402

p = configs.slab_problem(1)
b = P.build_rhs(p, device=True)
for restart in (30, None):
    P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=5, restart=restart))
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=6000, restart=restart))
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"restart={restart} its={rep.iterations} res={rep.true_residual:.3e} best={best * 1e3:.2f} ms "
          f"({best / rep.iterations * 1e6:.1f} us/it)")
